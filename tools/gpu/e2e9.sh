MESHREG_B200_DEBUG=2 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; grep -E "many|rep|batch_create|topolog|meshes|pixel|group" gpurun_out/e2e_dbg.log | tail -26
