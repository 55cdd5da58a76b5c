#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
for m in bench fused; do
  echo "== $m" >> ${O}_ab.log
  timeout -s KILL 1500 python tools/ab_variants.py run $m >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
done
echo done
