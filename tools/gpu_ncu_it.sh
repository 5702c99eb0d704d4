mkdir -p gpurun_out
for v in default pk; do
  if [ "$v" = default ]; then L=""; else L="variants/$v.so"; fi
  ILS_LIB=$L timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:'k_row|k_col2' --launch-skip 1 --launch-count 2 -o gpurun_out/it_$v python tools/time_u8.py --frames 1 > gpurun_out/ncu_it_$v.log 2>&1
done
true
