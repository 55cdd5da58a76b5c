#!/bin/bash
# bulk copies per row A/B (+ parity of each split variant). usage: <tag>
set -u
mkdir -p gpurun_out
for v in split2 split4; do
  RLVLA_LIB=paper_2602_05765_b200/variants/$v.so timeout -s KILL 600 python -m pytest tests/test_parity_logprob.py -m gpu -q -x > gpurun_out/$1_pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/$1_pytest_$v.log
done
bash tools/gpu_ab.sh $1 bench fused bwd
echo done
