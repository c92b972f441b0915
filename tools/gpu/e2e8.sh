for c in 0 32 15; do echo "chunk $c"; timeout 600 python tools/e2e_many.py 64 $c 2>&1 | grep -E "rep" | tail -2; done
MESHREG_B200_DEBUG=2 timeout 600 python tools/e2e_many.py 64 32 > gpurun_out/e2e_dbg.log 2>&1; grep -E "many" gpurun_out/e2e_dbg.log | tail -22
