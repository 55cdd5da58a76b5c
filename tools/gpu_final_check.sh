#!/bin/bash
# one GPU: smoke + the whole GPU suite + one bench line at HEAD. usage: <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "head=$(cat .head 2>/dev/null)" > ${O}_pytest.log
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs --timeout 900 >> ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout -s KILL 900 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
