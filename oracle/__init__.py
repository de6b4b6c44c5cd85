"""TEST INFRASTRUCTURE ONLY — CPU restatements of the reference GEMM path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import anything under oracle/.  The product package
(paper_1705_05249_b200) never does; its compute path is libtbgemm.so.
"""
