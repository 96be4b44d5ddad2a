set -x
PBAD_GPU_CHAIN_V6=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r2_c6_parity.log
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x -k C3 2>&1 | tail -5 >> gpurun_out/r2_c6_parity.log
for c in C3 C2; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/r2_c6_bench.log; done
PBAD_GPU_CHAIN_V6=1 timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/r2_c6_bench.log
