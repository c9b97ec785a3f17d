timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
LQG_CORESIDENT=1 timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -x -q 2>&1 | tail -2
for lib in variants/prev2.so paper_2509_01229_b200/liblqg.so; do
 for s in "8192 28672" "28672 8192"; do set -- $s
  for m in 256 1024 4096; do echo "$lib $1x$2: $(LQG_LIB_PATH=$lib timeout 60 python tools/profile_one.py --n $1 --k $2 --m $m --time 2>&1 | tail -1)"; done
 done
done
python tools/ab.py --libs variants/prev2.so,paper_2509_01229_b200/liblqg.so --ms 1,16,64,128,256,512,1024,2048,4096 --rounds 2 2>&1
