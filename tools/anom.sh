# intermittent join-phase stalls: phase probe repeated (allocator counters printed)
for i in 1 2 3 4 5 6; do python tools/phase_probe.py --config 5 --reps 10; done
for i in 1 2 3 4; do PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/phase_probe.py --config 5 --reps 10; done
