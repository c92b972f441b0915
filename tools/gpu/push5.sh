timeout 300 python tools/push_profile.py 64 c4 2>&1 | tail -10
timeout 300 python tools/push_profile.py 1 c2 2>&1 | tail -10
