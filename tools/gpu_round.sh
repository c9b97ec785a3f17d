# One GPU round of evidence: parity, smoke, bench (both arms), launch list,
# ncu --set full per LLaMA-2-70B layer shape at M = 16 and 4096, MoE timing.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
for s in "10240 8192" "8192 8192" "28672 8192" "8192 28672"; do
  set -- $s
  for m in 16 4096; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:lqg_w4a8 -s 2 -c 1 -o gpurun_out/prof_${1}x${2}_m$m python tools/profile_one.py --n $1 --k $2 --m $m > gpurun_out/prof_${1}x${2}_m$m.log 2>&1; echo "ncu $1x$2 m=$m rc=$?"
  done
done
timeout 300 python tools/moe_time.py > gpurun_out/moe_time.txt 2>&1; tail -10 gpurun_out/moe_time.txt
for m in 1 16 64 128 256 1024 4096; do timeout 120 python tools/profile_one.py --n 8192 --k 28672 --m $m --time; done
