D=paper_2509_01229_b200
LQG_LIB_PATH=$PWD/$D/liblqg_exp.so timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/ab.py --libs $D/liblqg.so,$D/liblqg_exp.so --ms 1,16,64,128,512,4096 --rounds 3
