for mv in 2048 1024 512 256; do echo "MINVOX $mv"; BQ_PROX_MINVOX=$mv timeout 120 python bench/micro/prox_small.py 2>&1 | tail -4 | cut -c1-60; done
