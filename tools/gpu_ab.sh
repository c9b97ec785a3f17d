timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/ab.py --libs variants/prev3.so,paper_2509_01229_b200/liblqg.so --ms 1,16,64,256,1024,4096 --rounds 2 2>&1
