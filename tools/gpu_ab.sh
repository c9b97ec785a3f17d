python -m pytest tests -m gpu -q -x 2>&1 | tail -3
P=paper_2509_01229_b200/liblqg.so
LQG_PAIR=0 python tools/moe_time.py 2>&1 | tail -12
python tools/moe_time.py 2>&1 | tail -12
