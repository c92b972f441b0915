for lib in paper_1411_2141_b200/libmeshreg_b200.so build_exp/libmrb_tg.so; do
  echo "== $lib"; MESHREG_B200_LIB=$PWD/$lib MESHREG_B200_DEBUG=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "exchange|^\{" | tail -2 | cut -c1-150
done
MESHREG_B200_LIB=$PWD/build_exp/libmrb_tg.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "golden" 2>&1 | tail -1
