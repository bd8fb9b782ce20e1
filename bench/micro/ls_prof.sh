set -x
NCU=/usr/local/cuda/bin/ncu
python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ls256_b8.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/ls256_launches.csv python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_l.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:zc_kernel -s 4 -c 1 -o gpurun_out/zc512 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_z512.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:zc_kernel -s 4 -c 1 -o gpurun_out/zc256 python bench/ls_bench.py --n 128 --views 16 --batch 16 --steps 1 > gpurun_out/ncu_z256.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:xi_kernel -s 4 -c 1 -o gpurun_out/xi512 python bench/ls_bench.py --n 256 --views 8 --batch 8 --steps 1 > gpurun_out/ncu_x512.log 2>&1
ls -la gpurun_out
