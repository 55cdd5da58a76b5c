#!/bin/bash
# 4-GPU call: multi-GPU parity (N = 2, 4; in-kernel P2P and NCCL) + weak-scaling bench at N = 2, 4.
# usage: tools/gpu_r2_mgpu.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
nvidia-smi topo -m > ${O}_topo.txt 2>&1
git_head=$(cat .head 2>/dev/null); echo "head=${git_head}" > ${O}_pytest.log
timeout -s KILL 900 python -m pytest tests/test_multigpu.py -v --timeout 400 >> ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
for N in 2 4; do
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N > ${O}_bench_n$N.log 2>&1; echo "rc=$?" >> ${O}_bench_n$N.log
done
echo done
