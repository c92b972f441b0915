timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "wave_groups or batch or pipelined" 2>&1 | tail -2
echo "== default nodebug"; timeout 600 python tools/e2e_many.py 64 0 2>&1 | grep -E "rep" | tail -2
echo "== no defer"; MESHREG_B200_NO_DEFER=1 timeout 600 python tools/e2e_many.py 64 0 2>&1 | grep -E "rep" | tail -2
MESHREG_B200_DEBUG=2 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; grep -E "many|rep" gpurun_out/e2e_dbg.log | tail -6
