#!/bin/bash
# A/B a BASELINE config's decode across library builds (GPU box):
#   tools/ab_cfg.sh "units s g m b ratio [tables]" libA.so libB.so [rounds]
CFG=$1; A=$2; B=$3; R=${4:-2}
for i in $(seq 1 $R); do
  for L in $A $B; do
    v=$(PQKV_LIB=$L timeout 300 python tools/prof_cfg5.py $CFG 2>/dev/null | grep "^decode" | sed 's/.*: \([0-9.]*\) us\/step.*/\1/')
    echo "$CFG $L $v"
  done
done
