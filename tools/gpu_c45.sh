mkdir -p gpurun_out
timeout 600 python tools/bench_c4.py > gpurun_out/c4.log 2>&1
timeout 600 python tools/bench_c5.py > gpurun_out/c5.log 2>&1
timeout 600 python tools/bench_c5.py --slab --check >> gpurun_out/c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -c 60 --csv --log-file gpurun_out/c4_launches.csv python tools/bench_c4.py --frames 4 > /dev/null 2>&1
true
