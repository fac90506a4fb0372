"""Launch footprints of the stall_gemm leg's prefill kernels (for ncu): one layer at 4K and 64K."""
import torch
from flash_attn import flash_attn_func
dev = torch.device("cuda", 0)
w = [torch.randn(k, n, dtype=torch.bfloat16, device=dev) * 0.01 for k, n in ((4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096))]
for ctx in (4096, 65536):
    cached = ctx * 7 // 8; m = ctx - cached
    x = torch.randn(m, 4096, dtype=torch.bfloat16, device=dev)
    k = torch.randn(1, cached, 8, 128, dtype=torch.bfloat16, device=dev)
    qkv = torch.matmul(x, w[0])
    q = qkv[:, :4096].view(1, m, 32, 128); kn = qkv[:, 4096:5120].view(1, m, 8, 128); vn = qkv[:, 5120:].view(1, m, 8, 128)
    a = flash_attn_func(q, k, k, causal=False) + flash_attn_func(q, kn, vn, causal=True)
    torch.matmul(a.view(m, 4096), w[1]); gu = torch.matmul(x, w[2]); torch.matmul(gu[:, :14336], w[3])
    torch.cuda.synchronize()
