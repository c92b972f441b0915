for c in 64 32 22 15; do echo "chunk $c"; MESHREG_B200_DEBUG= timeout 600 python tools/e2e_many.py 64 $c 2>&1 | grep "^rep" | tail -2; done
