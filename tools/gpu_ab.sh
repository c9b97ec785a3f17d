LQG_UA=1 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
P=paper_2509_01229_b200/liblqg.so
python tools/ab.py --libs $P,$P --env "LQG_UA=0;LQG_UA=1" --ms 1,16,32,64 --rounds 3
