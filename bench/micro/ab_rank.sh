# rank/size microbench for the in-tree lib and an A/B variant ($1), + prox parity with the variant
V=${1:-paper_2307_02043_b200/lib/ab/libbq_l4.so}
echo "== in-tree"; timeout 120 python bench/micro/prox_rank_sizes.py 2>&1 | tail -4
echo "== $V"; BQ_LIB=$V timeout 120 python bench/micro/prox_rank_sizes.py 2>&1 | tail -4
BQ_LIB=$V timeout 300 python -m pytest tests/test_prox_gpu.py -x -q 2>&1 | tail -2
