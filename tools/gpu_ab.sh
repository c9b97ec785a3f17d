P=paper_2509_01229_b200/liblqg.so
python tools/ab.py --libs $P,$P,$P --env "LQG_DEBUG_MAX_BN=192;LQG_DEBUG_MAX_BN=224;LQG_DEBUG_MAX_BN=208" --ms 1024,2048,4096,8192 --rounds 2
