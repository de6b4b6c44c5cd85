import os, sys, subprocess
for dbg in (0, 1, 2, 4, 3, 5, 6, 7):
    env = dict(os.environ, TBGEMM_DBG=str(dbg))
    out = subprocess.run([sys.executable, "tools/exp3.py"], env=env, capture_output=True, text=True).stdout
    for line in out.splitlines():
        if line.startswith("H"):
            print("dbg", dbg, line, flush=True)
