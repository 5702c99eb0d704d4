mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:'k_u8|k_row' -c 400 --csv --log-file gpurun_out/u8k.csv python tools/time_u8.py --frames 2 > /dev/null 2>&1
true
