echo "== default nodebug"; timeout 600 python tools/e2e_many.py 64 0 2>&1 | grep -E "rep" | tail -3
MESHREG_B200_DEBUG=1 timeout 600 python tools/e2e_many.py 64 0 > gpurun_out/e2e_dbg.log 2>&1; grep -E "many|rep|batch_create|topolog|meshes|pixel" gpurun_out/e2e_dbg.log | tail -20
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pixel.py -q -p no:cacheprovider -x 2>&1 | tail -2
