#!/bin/bash
# full GPU check (run with gpurun --gpus 4 so the multi-GPU parity cases run too):
# pytest -m gpu, smoke, bench N=1. usage: tools/gpu_r2_full.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "head=$(cat .head 2>/dev/null) gpus=$(nvidia-smi -L | wc -l)" > ${O}_pytest.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs --timeout 900 >> ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
echo done
