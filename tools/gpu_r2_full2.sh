#!/bin/bash
# 4 GPUs: full pytest -m gpu, smoke, bench N=1, flow A/B (24,576 and 196,608 steps)
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
echo "head=$(cat .head 2>/dev/null) gpus=$(nvidia-smi -L | wc -l)" > ${O}_pytest.log
timeout -s KILL 1800 python -m pytest tests -m gpu -q -rs --timeout 900 >> ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
timeout -s KILL 300 python __graft_entry__.py smoke > ${O}_smoke.log 2>&1; echo "smoke rc=$?" >> ${O}_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py > ${O}_bench.log 2>&1; echo "bench rc=$?" >> ${O}_bench.log
for rows in 24576 196608; do
  echo "== flow rows=$rows" >> ${O}_flow.log
  FLOW_ARGS="--rows $rows" CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python tools/ab_variants.py run flow >> ${O}_flow.log 2>&1
  echo "== flow learned f32 rows=$rows" >> ${O}_flow.log
  FLOW_ARGS="--rows $rows --learned --f32" CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python tools/ab_variants.py run flow >> ${O}_flow.log 2>&1
done
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python tools/prof_fused.py --mode fused --f32 --vocab 32000 --rows 32768 --iters 10 > ${O}_rowf32.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 300 python tools/prof_fused.py --mode fwd --f32 --vocab 32000 --rows 32768 --iters 10 >> ${O}_rowf32.log 2>&1
echo done
