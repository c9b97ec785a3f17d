LQG_CORESIDENT=1 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/ab.py --libs paper_2509_01229_b200/liblqg.so,paper_2509_01229_b200/liblqg.so,paper_2509_01229_b200/liblqg.so,paper_2509_01229_b200/liblqg.so --env ";LQG_CORESIDENT=1;LQG_CORESIDENT=1,LQG_L2_PREFETCH_CHUNKS=0;LQG_CORESIDENT=1,LQG_PDL_TRIGGER=0" --ms 1,16,32 --rounds 2 2>&1
