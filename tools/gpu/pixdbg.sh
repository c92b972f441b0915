CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/pix_dbg.py f32 64 64 1 0 0.0 2>&1 | tail -4
CUDA_LAUNCH_BLOCKING=1 MESHREG_B200_PIX_NOTMA=1 timeout 60 python tools/pix_dbg.py f32 64 64 1 3 0.8 2>&1 | tail -4
