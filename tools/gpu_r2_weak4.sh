#!/bin/bash
# 4 GPUs: multi-GPU parity tests + weak-scaling bench lines at N = 2, 4. usage: <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests/test_multigpu.py -m gpu -q -rs --timeout 600 > ${O}_pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest_mgpu.log
for n in 2 4; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n > ${O}${n}_bench.log 2>&1; echo "rc=$?" >> ${O}${n}_bench.log
done
echo done
