# attention A/B: parity tests + timing of the one-tile (HC_ATTN_TC=1) and two-tile kernels
timeout 600 python -m pytest tests/test_k6_blocks_gpu.py -q -x -k attention 2>&1 | tail -3
HC_ATTN_TC=1 timeout 300 python scripts/attn_probe.py 2>&1 | tail -4
timeout 300 python scripts/attn_probe.py 2>&1 | tail -4
