# A/B of the config-2 prox step between two builds: BQ_LIB=<old .so> vs the in-tree lib (alternating)
OLD=${1:-paper_2307_02043_b200/lib/ab/libbq_old.so}
for i in 1 2; do
  echo -n "old: "; BQ_LIB=$OLD python bench.py --no-ls --no-cpu --steps 60 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
  echo -n "new: "; python bench.py --no-ls --no-cpu --steps 60 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
