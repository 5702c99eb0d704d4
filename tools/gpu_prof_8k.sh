# ncu --set full of the first four passes (F0, col, IT, col) of one 8K RGB image
# (C5 geometry), summarised on the box, plus the SASS stall sources of IT and col
mkdir -p gpurun_out/prof
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_row|k_col' -s 9 -c 4 -o /tmp/seq_8k -f python tools/prof_smooth.py --frames 1 --h 4320 --w 7680 > gpurun_out/ncu_seq8k.log 2>&1
python tools/ncu_summary.py /tmp/seq_8k.ncu-rep gpurun_out/prof/seq_8k_summary.txt "one 8K RGB image" traffic_8k.json > /dev/null 2>&1
ncu -i /tmp/seq_8k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_col2 --launch-count 1 > /tmp/col8k.csv 2>/dev/null
python tools/ncu_sass_hot.py /tmp/col8k.csv --top 40 > gpurun_out/prof/col8k_hot.txt 2>&1
ncu -i /tmp/seq_8k.ncu-rep --page source --csv --print-source sass --kernel-name regex:k_row --launch-skip 1 --launch-count 1 > /tmp/it8k.csv 2>/dev/null
python tools/ncu_sass_hot.py /tmp/it8k.csv --top 40 > gpurun_out/prof/it8k_hot.txt 2>&1
ncu -i /tmp/seq_8k.ncu-rep --page details --csv > gpurun_out/prof/seq_8k_details.csv 2>/dev/null
true
