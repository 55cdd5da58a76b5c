#!/bin/bash
# NEXT-4 flow kernel: parity tests, then A/B of the TMA-staged variants (tools/ab_variants.py)
mkdir -p gpurun_out
O=gpurun_out/$1
timeout -s KILL 400 python -m pytest tests/test_parity_flow.py tests/test_fullsize.py -q -m gpu -k "flow" > ${O}_tests.log 2>&1
echo "tests rc=$?" >> ${O}_tests.log
timeout -s KILL 500 python tools/ab_variants.py run flow > ${O}_ab_bf16.log 2>&1
FLOW_ARGS="--learned --f32" timeout -s KILL 500 python tools/ab_variants.py run flow > ${O}_ab_f32l.log 2>&1
FLOW_ARGS="--rows 24576" timeout -s KILL 500 python tools/ab_variants.py run flow > ${O}_ab_small.log 2>&1
