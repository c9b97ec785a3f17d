# ncu --set full of one launch per LLaMA-2-70B layer shape at M = 16 and 4096,
# summarised on the box (reports are too large to ship back).
# SHAPES="n k;n k" and MS="m m" select other shapes / token counts (e.g. the
# LLaMA-2-7B shapes: SHAPES="12288 4096;4096 4096;22016 4096;4096 11008").
mkdir -p gpurun_out/ncu
IFS=";" read -ra SHAPE_LIST <<< "${SHAPES:-10240 8192;8192 8192;28672 8192;8192 28672}"
for s in "${SHAPE_LIST[@]}"; do
  set -- $s
  for m in ${MS:-16 4096}; do
    timeout 600 ncu --set full --clock-control none -k regex:lqg_w4a8 -s 2 -c 1 -o gpurun_out/ncu/prof_${1}x${2}_m$m python tools/profile_one.py --n $1 --k $2 --m $m > /dev/null 2>&1; echo "ncu $1x$2 m=$m rc=$?"
    B=$(python -c "n,k,m=$1,$2,$m; print(n*k//2+2*n*k//128+4*n+m*k+4*m+2*m*n)"); O=$(python -c "print(2*$m*$1*$2)")
    python tools/ncu_summary.py rep gpurun_out/ncu/prof_${1}x${2}_m$m.ncu-rep --bytes $B --ops $O > gpurun_out/r_ncu_${1}x${2}_m$m.json
    ncu -i gpurun_out/ncu/prof_${1}x${2}_m$m.ncu-rep --page details > gpurun_out/r_ncu_${1}x${2}_m$m.details.txt 2>&1
  done
done
python tools/ncu_summary.py traffic gpurun_out/ncu/prof_*x*_m*.ncu-rep > gpurun_out/${NCU_SUMMARY:-ncu_summary.json}
rm -rf gpurun_out/ncu
ls -la gpurun_out
