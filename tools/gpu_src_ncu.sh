# ncu source-level stall sampling of one launch: N K M
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --warp-sampling-interval ${NCU_SI:-auto} --clock-control none -k regex:lqg_w4a8 -s 2 -c 1 -o gpurun_out/src_$1x$2_m$3 python tools/profile_one.py --n $1 --k $2 --m $3 > gpurun_out/src_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/src_$1x$2_m$3.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1x$2_m$3.sass.csv 2>&1
ncu -i gpurun_out/src_$1x$2_m$3.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_$1x$2_m$3.cuda.csv 2>&1
ncu -i gpurun_out/src_$1x$2_m$3.ncu-rep --page details > gpurun_out/src_$1x$2_m$3.details.txt 2>&1
ls -la gpurun_out/src_*
