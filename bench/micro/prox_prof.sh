# bench line + launch list + one full ncu capture of the prox kernel and of the LS ZC pass (round profiles)
NCU=/usr/local/cuda/bin/ncu
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench.log | cut -c1-300
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
$NCU --set full --clock-control none --import-source on -k regex:wtv_fused_kernel -s 3 -c 1 -o gpurun_out/prof \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-ls > gpurun_out/ncu_full.log 2>&1; echo "full rc $?"
$NCU --set full --clock-control none --import-source on -k regex:zc_kernel -s 4 -c 1 -o gpurun_out/zc512 \
  python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_z512.log 2>&1; echo "zc rc $?"
