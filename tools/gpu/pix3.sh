timeout 900 python -m pytest tests/test_gpu_pixel.py -q -p no:cacheprovider > gpurun_out/pytest_pixel.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_pixel.log
timeout 300 python tools/pixel_bench.py 64 f32 100 2
timeout 300 python tools/pixel_bench.py 64 f64 100 2
timeout 300 python tools/pixel_bench.py 8 f32 100 2
