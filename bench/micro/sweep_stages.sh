for ns in 2 3 4; do for w in 15 12 10 8 6; do
  r=$(BQ_PROX_STAGES=$ns BQ_PROX_WARPS=$w timeout 60 python bench.py --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), round(d['prox_phases_last_step']['dual']['ms']*10,1), round(d['prox_phases_last_step']['newton']['ms'],3))")
  echo "stages=$ns warps=$w -> $r"
done; done
