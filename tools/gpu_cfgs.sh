#!/bin/bash
# 1-GPU: streamer parity test + bench on every BJ config that fits one GPU (micro-batched)
mkdir -p gpurun_out
O=gpurun_out/$1
export RLVLA_DEBUG=1
timeout -s KILL 600 python -m pytest tests/test_streamer.py tests/test_parity_path.py -m gpu -q --timeout 300 > ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
for c in libero_spatial_oft libero10_long maniskill_ppo_gae grpo_span; do
  timeout -s KILL 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > ${O}_bench_$c.log 2>&1; echo "rc=$?" >> ${O}_bench_$c.log
done
