# round-2 K6 captures: ncu --set full of the Q projection (N=4096 pair GEMM,
# tail-split last wave), the O projection, FC2 and the prefill attention of
# one 7B recompute layer (scripts/prof_k6.py: per call the pair launches are
# KV0 Q0 O0 FC1 FC2 KV1; 4 warm-up calls)
set -x
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o gpurun_out/$1 python scripts/prof_k6.py > gpurun_out/$1.log 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
}
cap r2_q_gemm tc_gemm_pair 25
cap r2_o_gemm tc_gemm_pair 26
cap r2_fc2_gemm tc_gemm_pair 28
cap r2_attn attn_fa 4
