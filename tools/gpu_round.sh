# One GPU round of evidence (part 1): parity, smoke, bench (both arms), launch
# list, MoE timing. Part 2 (tools/gpu_ncu.sh): ncu --set full per 70B shape.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/moe_time.py > gpurun_out/moe_time.txt 2>&1; tail -4 gpurun_out/moe_time.txt
timeout 300 python bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_gpus2.log 2>&1; echo "bench --gpus 2 on this box rc=$? (non-zero expected with one GPU)"; tail -2 gpurun_out/bench_gpus2.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.txt
done
