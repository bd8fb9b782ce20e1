# Round profiles: tests, bench line, launch list of the same command, one full ncu capture of the
# prox kernel, LS launch lists (n=128 16 views, n=256 8 views) and a full capture of ZC.
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gpu tests rc $?"; tail -2 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-more > gpurun_out/plain_launch.log 2>&1 &&
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-more > gpurun_out/ncu_launch.log 2>&1; echo "launch rc $?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-ls --no-more > gpurun_out/plain_full.log 2>&1 &&
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:wtv_fused_kernel -s 3 -c 1 -o gpurun_out/prof \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-ls --no-more > gpurun_out/ncu_full.log 2>&1; echo "full rc $?"
timeout 600 python bench/ls_bench.py --n 128 --views 16 --batch 16 --steps 1 > gpurun_out/plain_l128.log 2>&1 &&
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/ls128_launches.csv python bench/ls_bench.py --n 128 --views 16 --batch 16 --steps 1 > gpurun_out/ncu_l128.log 2>&1; echo "ls128 rc $?"
timeout 600 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/plain_l256.log 2>&1 &&
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ls256_launches.csv python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_l256.log 2>&1; echo "ls256 rc $?"
