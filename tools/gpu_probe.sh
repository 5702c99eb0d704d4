mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:k_row -c 300 --csv --log-file gpurun_out/u8_launches.csv python tools/time_u8.py --frames 2 > /dev/null 2>&1
true
