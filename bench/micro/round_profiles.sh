# Round profiles: bench line, launch list of the same command, one full ncu capture of the
# prox kernel, LS launch lists (n=128 16 views, n=256 8 views) and full captures of ZC.
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-more > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:wtv_fused_kernel -s 3 -c 1 -o gpurun_out/prof \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-ls --no-more > gpurun_out/ncu_full.log 2>&1; echo "full rc $?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/ls128_launches.csv python bench/ls_bench.py --n 128 --views 16 --batch 16 --steps 1 > gpurun_out/ncu_l128.log 2>&1; echo "ls128 rc $?"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ls256_launches.csv python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_l256.log 2>&1; echo "ls256 rc $?"
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:zc_kernel -s 4 -c 1 -o gpurun_out/zc256 \
  python bench/ls_bench.py --n 128 --views 16 --batch 16 --steps 1 > gpurun_out/ncu_z256.log 2>&1; echo "zc rc $?"
timeout 900 python bench/ls_bench.py --n 256 --views 120 --batch 30 --steps 1 > gpurun_out/ls256_full.log 2>&1; echo "ls256 full rc $?"
