timeout 300 python tools/phase_profile.py 8 c4
timeout 300 python tools/phase_profile.py 1 c2
