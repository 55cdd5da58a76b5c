#!/bin/bash
# multi-GPU call: NCCL parity + bench at N = $2
mkdir -p gpurun_out
O=gpurun_out/$1
N=$2
export RLVLA_DEBUG=1
nvidia-smi topo -m > ${O}_topo.txt 2>&1
timeout -s KILL 400 python -m pytest tests/test_multigpu.py -q --timeout 300 -x > ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N > ${O}_bench.log 2>&1; echo "rc=$?" >> ${O}_bench.log
