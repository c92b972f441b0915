for env in "MESHREG_B200_NPT=1" "MESHREG_B200_NPT=1 MESHREG_B200_EXCHANGE=pull" "MESHREG_B200_NPT=2 MESHREG_B200_EXCHANGE=pull"; do
  echo "== $env"; env $env MESHREG_B200_DEBUG=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "exchange|^\{" | tail -2 | cut -c1-150
done
