LQG_SKEW=16 python -m pytest tests/test_gemm_gpu.py tests/test_grouped_gpu.py -q -x 2>&1 | tail -2
P=paper_2509_01229_b200/liblqg.so
python tools/ab.py --libs $P,$P,$P,$P --env "LQG_SKEW=0;LQG_SKEW=8;LQG_SKEW=16;LQG_SKEW=32" --ms 1,16,64,128 --rounds 2
