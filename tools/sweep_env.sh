#!/bin/bash
# usage: tools/sweep_env.sh VAR "v1 v2 ..." cfg...   (quick per-config stage timings for each value)
var=$1; vals=$2; shift 2
for v in $vals; do
  echo "== $var=$v"
  env $var=$v bash tools/bench_gather.sh "$@"
done
