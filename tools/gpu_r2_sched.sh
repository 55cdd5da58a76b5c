#!/bin/bash
# schedule A/B + streamer tests + verbose multi-GPU logs. usage: tools/gpu_r2_sched.sh <tag>
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 600 python -m pytest tests/test_streamer.py -q -rs --timeout 300 > ${O}_streamer.log 2>&1; echo "rc=$?" >> ${O}_streamer.log
for sch in "serial" "pipelined --reserve-sms 0" "pipelined --reserve-sms 1" "pipelined --reserve-sms 2" "pipelined --reserve-sms 4"; do
  echo "== $sch" >> ${O}_bench.log
  CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python bench.py --schedule $sch --no-cpu-baseline --trace gpurun_out/$1_trace_${sch// /_}.json >> ${O}_bench.log 2>&1; echo "rc=$?" >> ${O}_bench.log
done
if [ "$(nvidia-smi -L | wc -l)" -ge 4 ]; then
  for mode in p2p-only; do for n in 4 8; do
    RLVLA_MGPU_MODE=$mode timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tools/mgpu_parity.py > ${O}_mgpu_${mode}_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_${mode}_n$n.log
  done; done
  for n in 2 4; do
    timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n tools/mgpu_parity.py > ${O}_mgpu_nccl-p2p_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_nccl-p2p_n$n.log
    RLVLA_P2P=0 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n tools/mgpu_parity.py > ${O}_mgpu_nccl_n$n.log 2>&1; echo "rc=$?" >> ${O}_mgpu_nccl_n$n.log
    timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n > ${O}_bench_n$n.log 2>&1; echo "rc=$?" >> ${O}_bench_n$n.log
  done
fi
echo done
