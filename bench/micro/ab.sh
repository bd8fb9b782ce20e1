# A/B of the config-2 prox (and the prox_more shapes) between builds, alternating in ONE call
# (boxes differ by a few %): bash bench/micro/ab.sh base [other tags...]; "cur" = the in-tree lib
pr='import json,sys; d=json.loads(sys.stdin.read()); p=d["prox_phases_last_step"]; print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), "fused", p["fused"]["ms"], "work", p["fused"]["work_ms"], "nloc", p["newton_local"]["ms"], "nfull", p["newton_full"]["ms"], [round(q["ms_per_solve"],3) for q in d.get("prox_more",[])])'
for rep in 1 2; do
  for tag in "$@" cur; do
    lib=paper_2307_02043_b200/lib/ab/libbq_$tag.so
    [ $tag = cur ] && lib=paper_2307_02043_b200/lib/libbq.so
    echo -n "$tag: "; BQ_LIB=$lib python bench.py --no-ls --no-cpu --steps 40 ${AB_ARGS} 2>&1 | tail -1 | python -c "$pr"
  done
done
