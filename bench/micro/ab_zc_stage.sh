set -x
timeout 600 python -m pytest tests/test_ls_fft_gpu.py tests/test_physics_gpu.py -x -q 2>&1 | tail -2
for lib in "" paper_2307_02043_b200/lib/ab/libbq_nostg.so paper_2307_02043_b200/lib/ab/libbq_stg512.so; do
  echo "== lib=$lib"
  BQ_LIB=$lib timeout 300 python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
  BQ_LIB=$lib timeout 300 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 2>&1 | tail -1
done
BQ_LIB=paper_2307_02043_b200/lib/ab/libbq_stg512.so timeout 600 python -m pytest tests/test_ls_fft_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-ls --no-more --no-loop 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
