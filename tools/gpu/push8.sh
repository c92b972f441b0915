MESHREG_B200_EXCHANGE=push timeout 300 python tools/push_profile.py 64 c4 2>&1 | tail -9
