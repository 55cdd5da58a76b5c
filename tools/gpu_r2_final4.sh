#!/bin/bash
# round-2 evidence, 4 GPUs: pytest -m gpu (incl. multi-GPU parity), kept multi-GPU parity logs
# (2/4 ranks NCCL+P2P and NCCL, 4/8 ranks P2P-only), weak scaling N=2/4, strong scaling of the
# BASELINE configs quoted at a GPU count. usage: tools/gpu_r2_final4.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "head=$(cat .head 2>/dev/null) gpus=$(nvidia-smi -L | wc -l)" > ${O}_pytest.log
timeout -s KILL 2400 python -m pytest tests -m gpu -q -rs --timeout 900 >> ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
nvidia-smi topo -m > ${O}_topo.txt 2>&1
for n in 2 4; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n tools/mgpu_parity.py > ${O}_mgpu_nccl-p2p_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_nccl-p2p_n$n.log
  RLVLA_P2P=0 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n tools/mgpu_parity.py > ${O}_mgpu_nccl_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_nccl_n$n.log
done
for n in 4 8; do
  RLVLA_MGPU_MODE=p2p-only timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tools/mgpu_parity.py > ${O}_mgpu_p2p-only_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_p2p-only_n$n.log
done
for n in 2 4; do
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n > ${O}${n}_bench.log 2>&1; echo "rc=$?" >> ${O}${n}_bench.log
done
bash tools/gpu_strong.sh $1_strong > ${O}_strong_rc.log 2>&1
echo done
