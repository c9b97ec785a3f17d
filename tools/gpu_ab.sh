P=paper_2509_01229_b200/liblqg.so
python tools/ab.py --libs $P,$P,$P,$P,$P --env "LQG_DEBUG_STAGES=16;LQG_DEBUG_STAGES=8;LQG_DEBUG_STAGES=6;LQG_DEBUG_STAGES=4;LQG_DEBUG_STAGES=3" --ms 16,64,128 --rounds 2
