# A/B of the LS subset gradient between builds (alternating, one call): bash bench/micro/ab_ls.sh "<tags>" [n views batch]
tags=$1; n=${2:-256}; views=${3:-8}; batch=${4:-8}
for rep in 1 2; do
  for t in $tags cur; do
    lib=paper_2307_02043_b200/lib/ab/libbq_$t.so
    [ $t = cur ] && lib=paper_2307_02043_b200/lib/libbq.so
    echo -n "$t: "; BQ_LIB=$lib python bench/ls_bench.py --n $n --views $views --batch $batch --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms'],2), 'ms', round(d['achieved_GBps']), 'GB/s', d['K_f'], d['K_a'], d['grad_norm'])"
  done
done
