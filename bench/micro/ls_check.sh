python -m pytest tests/test_ls_fft_gpu.py tests/test_physics_gpu.py -x -q 2>&1 | tail -3
python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 2>&1 | tail -1
