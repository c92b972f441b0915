for v in "IT=1 PASSES=1" "IT=25 PASSES=1"; do echo "== $v"; env $v MESHREG_B200_CS=16 timeout 20 python tools/push_dbg.py single gen64 2>&1 | grep -E "ok|rror" | tail -1; done
