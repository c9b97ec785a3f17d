python tools/trace_seq.py 16 2>&1 | tee gpurun_out/trace_seq16.txt
python tools/trace.py 8192x28672x16 4 2>&1 | tee gpurun_out/trace_down16.txt
python tools/trace.py 8192x8192x16 4 2>&1 | tee gpurun_out/trace_o16.txt
LQG_DEBUG_NO_PDL=1 python tools/ab.py --libs paper_2509_01229_b200/liblqg.so --ms 1,16 --rounds 1 2>&1 | tail -3
python tools/ab.py --libs paper_2509_01229_b200/liblqg.so --ms 1,16 --rounds 1 2>&1 | tail -3
