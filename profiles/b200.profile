# NVIDIA B200 (sm_100a, 148 SMs) device profile for the reference's analytic
# cost model (lq::parse_profile, cost_model.hpp:53-58; src/cost_model.cpp),
# from numbers MEASURED on this pool's B200s rather than the datasheet:
#   mem_bw_bytes_per_s  6.463e12  device copy bandwidth (MEASURED_PEAKS.json hbm_gbs,
#                                 b.copy_(a) over 2 GiB, read+write bytes)
#   tc_int8_ops_per_s   3.051e15  cuBLASLt IMMA int8 8192^3 burst (profiles/int8_peak.json)
#   tc_fp16_ops_per_s   1.686e15  cuBLAS bf16 8192^3 burst (MEASURED_PEAKS.json bf16_tflops)
#   cuda_ops_per_s      3.72e13   scalar INT32 pipe: 148 SMs x 128 lanes x 1.965 GHz
#   max_blocks_per_sm   1         lqg runs one 448-thread CTA per SM (lqg_gemm.cuh)
# Diagnostics (tools/cost_model.py): transition batch M* = 118 for W4A8, i.e.
# HBM-bound below ~120 tokens and INT8-tensor-bound above, which the measured
# M sweep reproduces (profiles/r01_bench.jsonl).
name = b200-sxm-measured
mem_bw_bytes_per_s = 6.463e12
cuda_ops_per_s = 3.72e13
tc_int8_ops_per_s = 3.051e15
tc_fp16_ops_per_s = 1.686e15
num_sms = 148
max_blocks_per_sm = 1
