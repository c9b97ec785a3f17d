P=paper_2509_01229_b200/liblqg.so
python tools/ab.py --libs $P,$P,$P,$P --env "LQG_DEBUG_MAX_BN=192;LQG_DEBUG_MAX_BN=128;LQG_DEBUG_MAX_BN=96;LQG_DEBUG_MAX_BN=64" --ms 64,128,192,256 --rounds 2
