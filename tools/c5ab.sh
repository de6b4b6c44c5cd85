for i in 1 2; do
python bench.py --workload hgemm_c5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('new', d['ms_per_step'], d['value'], d['config'].get('kernel'), d['clocks']['sm_mhz'])"
TBGEMM_LIB=$PWD/paper_1705_05249_b200/_lib/libtbgemm_old.so python bench.py --workload hgemm_c5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('old', d['ms_per_step'], d['value'], d['config'].get('kernel'), d['clocks']['sm_mhz'])"
done
