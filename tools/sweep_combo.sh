#!/bin/bash
# usage: tools/sweep_combo.sh CFG "VAR1=a VAR2=b" "VAR1=c" ...   (one bench_gather line per env combo)
cfg=$1; shift
for combo in "$@"; do
  echo "== $combo"
  env $combo bash tools/bench_gather.sh $cfg
done
