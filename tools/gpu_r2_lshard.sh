#!/bin/bash
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
for n in 2 4 8; do
  /usr/bin/time -f "wall %e s" timeout -s KILL 900 env RLVLA_MGPU_MODE=p2p-only python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n tools/mgpu_parity.py > ${O}_lshard_n$n.log 2>&1; echo "rc=$?" >> ${O}_lshard_n$n.log
done
timeout -s KILL 1200 python -m pytest tests/test_multigpu.py -q -rs --timeout 900 > ${O}_pytest.log 2>&1; echo "rc=$?" >> ${O}_pytest.log
echo done
