MESHREG_B200_CS=16 IT=1 PASSES=1 timeout 30 python tools/push_trace.py gen64 2>&1 | head -2
for v in "IT=25 PASSES=1" "IT=25 PASSES=0"; do echo "== $v"; env $v MESHREG_B200_CS=16 timeout 20 python tools/push_dbg.py single gen64 2>&1 | grep -E "ok|rror" | tail -1; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -x 2>&1 | tail -2
