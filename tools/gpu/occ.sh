MESHREG_B200_DEBUG=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "candidate|cluster " | head -20
nvidia-smi -q | grep -i -E "gpc|multiprocessor" | head
for cs in 8 10; do MESHREG_B200_CS=$cs timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-140; done
