#!/bin/bash
# A/B of two builds of libtbgemm.so on one bench workload, ABBA order.
# usage: tools/lib_ab.sh WORKLOAD OLD_SO [rounds]
W=${1:-hgemm}; OLD=$2; R=${3:-3}
one() {
  TBGEMM_LIB=$1 python bench.py --workload $W --steps 20 --warmup 5 --no-extra --no-cpu-baseline 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$2', d['ms_per_step'], round(d['value']), d['roofline'].get('kernel'), d['clocks']['sm_mhz'])"
}
NEW=$PWD/paper_1705_05249_b200/_lib/libtbgemm.so
for i in $(seq $R); do
  one $NEW new; one $OLD old; one $OLD old; one $NEW new
done
