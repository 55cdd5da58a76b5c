#!/bin/bash
# strong scaling of the BASELINE configs quoted at a GPU count (fixed global envs split over N)
mkdir -p gpurun_out
O=gpurun_out/$1
for cfg in libero10_long grpo_span maniskill_ppo_gae; do
  for N in 1 2 4; do
    if [ $N -eq 1 ]; then
      timeout -s KILL 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > ${O}_${cfg}_n1.log 2>&1
    else
      timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --config $cfg --steps 10 --warmup 3 > ${O}_${cfg}_n$N.log 2>&1
    fi
    echo "$cfg N=$N rc=$?"
  done
done
