#!/bin/bash
# 1-GPU: selected tests (args after the tag) + smoke + default bench. usage: tools/gpu_r2_quick.sh <tag> [pytest targets...]
set -u
mkdir -p gpurun_out
O=gpurun_out/$1; shift
if [ $# -gt 0 ]; then
  timeout -s KILL 1200 python -m pytest "$@" -q -rs --timeout 600 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
fi
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout -s KILL 900 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
echo done
