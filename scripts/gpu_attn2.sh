timeout 900 python -m pytest tests/test_recompute_gpu.py tests/test_k6_blocks_gpu.py tests/test_forward_gpu.py tests/test_restore_gpu.py -x -q -m gpu 2>&1 | tail -2
echo base; HC_LIB_PATH=$PWD/scripts/_base/lib_base.so timeout 300 python scripts/prof_k6.py
echo new; timeout 300 python scripts/prof_k6.py
