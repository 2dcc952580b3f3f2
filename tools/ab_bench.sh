#!/bin/bash
# A/B the decode bench across library builds: tools/ab_bench.sh libA.so libB.so [rounds]
# (run on the GPU box; prints value per run)
A=$1; B=$2; R=${3:-2}
for i in $(seq 1 $R); do
  for L in $A $B; do
    v=$(PQKV_LIB=$L timeout 600 python bench.py --no-cpu-baseline --steps 300 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['attend_only']['ms']*1e3,2))")
    echo "$L $v"
  done
done
