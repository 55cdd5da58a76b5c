#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests/test_parity_logprob.py tests/test_parity_next2.py tests/test_guard_regions.py -q --timeout 600 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
for m in fused32 fwd32 bwd32; do
  echo "== $m" >> ${O}_ab.log
  timeout -s KILL 900 python tools/ab_variants.py run $m >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
done
echo done
