mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_requests_op_write.sum --cache-control none --clock-control none -k regex:'k_row|k_u8' -c 400 --csv --log-file gpurun_out/u8_launches.csv python tools/time_u8.py --frames 2 > /dev/null 2>&1
true
