timeout 900 python -m pytest tests/test_gpu_pixel.py -q -p no:cacheprovider > gpurun_out/pytest_pixel.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pixel.log
timeout 300 python tools/pixel_bench.py 64 f32 20 1 > gpurun_out/pix_plain.log 2>&1 && cat gpurun_out/pix_plain.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pixel_iter -s 5 -c 1 -o gpurun_out/prof_pix python tools/pixel_bench.py 64 f32 20 1 > gpurun_out/ncu_pix.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_pix.log
