LQG_PAIR=1 timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q -k "pair or llama" 2>&1 | tail -2
for env in "LQG_PAIR=0" "LQG_PAIR=1"; do
 for s in "8192 28672" "28672 8192"; do set -- $s
  for m in 1024 4096; do echo "$env $1x$2: $(env $env timeout 60 python tools/profile_one.py --n $1 --k $2 --m $m --time 2>&1 | tail -1)"; done
 done
done
