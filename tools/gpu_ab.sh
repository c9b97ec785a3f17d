timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for env in "LQG_DYN=0" "LQG_DYN=1" "LQG_DYN=1 LQG_DYN_UNITS_PER_SM=4"; do
 for shp in "--n 8192 --k 28672" "--n 8192 --k 8192"; do
  echo "$env $shp: $(env $env timeout 60 python tools/profile_one.py $shp --m 16 --time 2>&1 | tail -1)"
 done
done
python tools/ab.py --libs variants/base.so,paper_2509_01229_b200/liblqg.so,paper_2509_01229_b200/liblqg.so,paper_2509_01229_b200/liblqg.so --env ";;LQG_DYN_UNITS_PER_SM=4;LQG_DYN_UNITS_PER_SM=16" --ms 1,16,32 --rounds 1 2>&1
