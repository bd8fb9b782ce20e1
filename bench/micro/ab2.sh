pr='import json,sys; d=json.loads(sys.stdin.read()); p=d["prox_phases_last_step"]; print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), "fused", p["fused"]["ms"], "work", p["fused"]["work_ms"], "nloc", p["newton_local"]["ms"], [round(q["ms_per_solve"],3) for q in d.get("prox_more",[])])'
for rep in 1 2; do
  echo -n "base: "; BQ_LIB=paper_2307_02043_b200/lib/ab/libbq_base.so python bench.py --no-ls --no-cpu --steps 40 2>&1 | tail -1 | python -c "$pr"
  echo -n "cur nocl: "; BQ_PROX_NOCL=1 python bench.py --no-ls --no-cpu --steps 40 2>&1 | tail -1 | python -c "$pr"
  echo -n "cur: "; python bench.py --no-ls --no-cpu --steps 40 2>&1 | tail -1 | python -c "$pr"
done
