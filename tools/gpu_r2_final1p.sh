#!/bin/bash
# one GPU: the whole GPU test suite, then tools/gpu_r2_final1.sh (evidence). usage: <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "gpus=$(nvidia-smi -L | wc -l)" > ${O}_pytest.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -rs --timeout 900 >> ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
bash tools/gpu_r2_final1.sh $1
