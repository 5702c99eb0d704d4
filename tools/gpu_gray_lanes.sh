# gray legs (C1 512^2, C2 1080p): concurrent lanes
for l in 2 3 4 6 8 12 16; do ILS_GRAY_LANES=$l python bench.py --steps 5 --no-cpu --no-cufft --no-e2e --no-c4 --no-c5 --no-dropin 2>&1 | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($l, d['c1']['value'], d['c2']['value'])"; done
