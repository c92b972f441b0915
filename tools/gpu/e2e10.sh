# e2e timeline of mrb_register_many (C4), host + device events
MESHREG_B200_DEBUG=1 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; tail -60 gpurun_out/e2e_dbg.log
