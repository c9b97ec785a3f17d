# One build->measure iteration on the GPU box: the GPU parity suite, then the
# 70B per-M sweep (and optional knob variants passed as arguments).
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -${TAIL:-4}
timeout 300 python tools/sweep.py --ms ${MS:-1,16,64,128,256,1024,4096} ${SWEEP_ARGS} 2>&1 | tail -20
for t in "$@"; do echo "== tune $t"; timeout 300 python tools/sweep.py --ms ${MS:-1,16,64,128,256,1024,4096} --tune "$t" 2>&1 | tail -20; done
