#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 600 python -m pytest tests/test_parity_flow.py -q --timeout 300 > ${O}_fpytest.log 2>&1; echo "rc=$?" >> ${O}_fpytest.log
for args in "--rows 24576" "--rows 24576 --learned --f32" "--rows 196608" "--rows 196608 --learned --f32" "--rows 4096 --D 35"; do
  echo "== flow $args" >> ${O}_flow.log
  FLOW_ARGS="$args" timeout -s KILL 900 python tools/ab_variants.py run flow >> ${O}_flow.log 2>&1
done
echo done
