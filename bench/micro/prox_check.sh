# prox parity tests + rank/size microbench
python -m pytest tests/test_prox_gpu.py -x -q 2>&1 | tail -3
python bench/micro/prox_rank_sizes.py 2>&1 | tail -4
