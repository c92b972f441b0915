for args in "--pairs 64" "--pairs 60" "--pairs 4"; do echo "== $args"; timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['path'])"; done
echo "== 4 pairs NPT=1"; MESHREG_B200_NPT=1 timeout 300 python bench.py --pairs 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['path'])"
