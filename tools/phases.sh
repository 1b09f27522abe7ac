# per-phase device times (tools/phase_probe.py) for configs 2 3 5 (+4 with PHASES_ALL=1), then the GPU tests
mkdir -p gpurun_out
tag=${1:-ph}
cfgs="2 3 5"; [ -n "$PHASES_ALL" ] && cfgs="2 3 4 5"
for c in $cfgs; do python tools/phase_probe.py --config $c; done > gpurun_out/${tag}_phases.txt 2>&1
cat gpurun_out/${tag}_phases.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
