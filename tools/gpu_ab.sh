python bench.py > gpurun_out/bench_pair.log 2> gpurun_out/bench_pair.err; tail -c 300 gpurun_out/bench_pair.err
