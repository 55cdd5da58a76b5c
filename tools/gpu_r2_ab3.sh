#!/bin/bash
# parity of the log-prob kernels + A/B (fused) + base-clock timing of the current fused kernel
set -u
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 900 python -m pytest tests/test_parity_logprob.py tests/test_parity_next2.py tests/test_fullsize.py tests/test_guard_regions.py tests/test_parity_path.py tests/test_streamer.py -q -x --timeout 600 > ${O}_pytest.log 2>&1; echo "pytest rc=$?" >> ${O}_pytest.log
echo "== fused" >> ${O}_ab.log
timeout -s KILL 900 python tools/ab_variants.py run fused >> ${O}_ab.log 2>&1; echo "rc=$?" >> ${O}_ab.log
for v in base norf prev; do
  RLVLA_LIB=paper_2602_05765_b200/variants/$v.so timeout -s KILL 600 ncu --clock-control base --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:lp_ -s 1 -c 1 --csv python tools/prof_fused.py --mode fused --iters 1 > ${O}_base_$v.csv 2>&1
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:lp_rf -s 1 -c 1 -o ${O}_rf python tools/prof_fused.py --mode fused --iters 1 > ${O}_ncu_full.log 2>&1; echo "rc=$?" >> ${O}_ncu_full.log
echo done
