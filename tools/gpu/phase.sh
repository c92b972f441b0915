MESHREG_B200_DEBUG=1 timeout 300 python tools/phase_profile.py 64 c4 2>&1 | grep -v candidate | tail -25
