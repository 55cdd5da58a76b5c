set -u
mkdir -p gpurun_out
RLVLA_LIB=paper_2602_05765_b200/variants/dxbulk.so timeout -s KILL 900 python -m pytest tests/test_parity_logprob.py tests/test_streamer.py tests/test_parity_path.py -m gpu -x -q > gpurun_out/dxb_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/dxb_pytest.log
bash tools/gpu_ab.sh dxb fused bwd bench fused base:fused
