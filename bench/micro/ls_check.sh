# LS pass parity + config-4 / n=256 timings (optionally a second build variant: $1 = extra nvcc flags)
timeout 600 python -m pytest tests/test_ls_fft_gpu.py tests/test_physics_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
timeout 300 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 2>&1 | tail -1
if [ -n "$1" ]; then
  touch paper_2307_02043_b200/csrc/ls_fft.cu
  BQ_NVCC_EXTRA="$1" python -m paper_2307_02043_b200.build 2>&1 | tail -1
  timeout 300 python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
  timeout 300 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 2>&1 | tail -1
fi
