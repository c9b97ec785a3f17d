python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py > gpurun_out/bench_pair.log 2> gpurun_out/bench_pair.err; tail -c 3000 gpurun_out/bench_pair.log
