timeout 600 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -5
python tools/ab.py --libs variants/prev2.so,paper_2509_01229_b200/liblqg.so --ms 1,16,256,4096 --rounds 2 2>&1
