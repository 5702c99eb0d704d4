# ncu: column solve kernels k_col3 (default) vs k_col2 (ILS_COL3_SPEC=-1), 1080p RGB, one launch each
mkdir -p gpurun_out
for spec in -2 -1; do
  ILS_COL3_SPEC=$spec timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:'k_col' --launch-skip 1 --launch-count 1 -o gpurun_out/col_$spec python tools/time_u8.py --frames 1 > gpurun_out/ncu_col_$spec.log 2>&1
done
true
