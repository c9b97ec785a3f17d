set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
for m in 16 4096; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lqg_w4a8 -s 2 -c 1 -o gpurun_out/prof_down_m$m python tools/profile_one.py --n 8192 --k 28672 --m $m > gpurun_out/prof_$m.log 2>&1; echo "ncu m=$m rc=$?"
done
for m in 1 16 64 256 1024 4096; do timeout 120 python tools/profile_one.py --n 8192 --k 28672 --m $m --time; done
