# e2e device timeline of mrb_register_many (C4), host stamps without syncs
MESHREG_B200_DEBUG=2 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; tail -42 gpurun_out/e2e_dbg.log
