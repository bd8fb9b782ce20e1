# ZC view-group A/B (LS_ZC_VG = 1 / 2 / 4) + prox and LS parity + the bench line
timeout 900 python -m pytest tests/test_prox_gpu.py tests/test_ls_fft_gpu.py -x -q 2>&1 | tail -2
for lib in "" paper_2307_02043_b200/lib/ab/libbq_vg2.so paper_2307_02043_b200/lib/ab/libbq_vg4.so; do
  echo "== lib=$lib"
  BQ_LIB=$lib timeout 300 python bench/ls_bench.py --n 128 --views 64 --batch 16 --steps 2 2>&1 | tail -1
  BQ_LIB=$lib timeout 300 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 2>&1 | tail -1
done
BQ_LIB=paper_2307_02043_b200/lib/ab/libbq_vg2.so timeout 600 python -m pytest tests/test_ls_fft_gpu.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-ls --no-loop 2>&1 | tail -1 > gpurun_out/bench_ab2.json
python -c "import json; d=json.load(open('gpurun_out/bench_ab2.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['serial_ms_per_step'], [round(m['ms_per_solve'],3) for m in d['prox_more']], d['prox_phases_last_step'])"
