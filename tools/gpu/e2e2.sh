MESHREG_B200_DEBUG=1 timeout 600 python tools/e2e_breakdown.py 64 2>&1 | grep -v candidate | tail -30
