# K6 GEMM tile width: 256-column pair tiles only (HC_PAIR_BN=256) vs the
# per-GEMM choice (192 where its last wave wastes less), interleaved
timeout 900 python -m pytest tests/test_recompute_gpu.py tests/test_restore_gpu.py tests/test_k6_blocks_gpu.py tests/test_forward_gpu.py -q -x -m gpu 2>&1 | tail -3
for i in 1 2; do
  echo "256: $(HC_PAIR_BN=256 timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_bn256.json 2>&1 | tail -1)"
  echo "auto: $(timeout 300 python scripts/k6_breakdown.py --out gpurun_out/k6_bnauto.json 2>&1 | tail -1)"
done
