# end-of-session validation: the driver's round-end commands, twice for flakiness
mkdir -p gpurun_out
: > gpurun_out/final.log
for i in 1 2; do
  timeout 900 python -m pytest tests -m gpu -x -q >> gpurun_out/final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/final.log 2>&1
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu --no-cufft >> gpurun_out/final.log 2>&1
done
true
