# BiCGSTAB x/r update with 16-byte complex64 pairs vs HEAD's lib (lib/ab/libbq_head.so)
timeout 600 python -m pytest tests/test_ls_fft_gpu.py tests/test_physics_gpu.py -x -q 2>&1 | tail -1
for rep in 1 2; do
for lib in "" paper_2307_02043_b200/lib/ab/libbq_head.so; do
  echo "== lib=$lib"
  BQ_LIB=$lib timeout 300 python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
done
done
