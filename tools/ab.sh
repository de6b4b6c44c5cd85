#!/bin/bash
# A/B builds of libtbgemm.so on the same box: LIBS="old new" tools/ab.sh <workload...>
LIBS=${LIBS:-"old new"}
for rep in 1 2; do
for lib in $LIBS; do
  for w in "$@"; do
    TBGEMM_LIB=ab/$lib.so python bench.py --workload $w --steps 30 --warmup 5 --no-extra --no-cpu-baseline | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$w', round(d['ms_per_step']*1e3,1), 'us', d['roofline']['frac'])"
  done
done
done
