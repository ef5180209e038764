cd scripts
cat > /tmp/one.py <<'PY'
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd() + "/..")
import torch
from paper_2410_05004_b200.capi import check, lib
s = torch.cuda.current_stream().cuda_stream
m, n, k = 16, 4096, 4096
a = torch.randn(m, k, device="cuda").bfloat16(); b = torch.randn(n, k, device="cuda").bfloat16()
x = torch.zeros(m, n, device="cuda"); xb = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    check(lib().hc_gemm_epilogue(1, a.data_ptr(), b.data_ptr(), m, n, k, x.data_ptr(), xb.data_ptr(), None, None, None, 0, s))
torch.cuda.synchronize()
PY
ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 3 -c 1 -o ../gpurun_out/skinny python /tmp/one.py > ../gpurun_out/skinny.log 2>&1
tail -3 ../gpurun_out/skinny.log
