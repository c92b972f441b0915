timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for w in c2 c1; do for p in "" grid; do echo "== $w $p"; MESHREG_B200_PATH=$p timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-120; done; done
