"""Probe: vLLM's vendored FlashAttention-4 (CuTe DSL, sm100) vs cuDNN SDPA vs ours at the bench shape."""
import math
import sys
import time

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, ".")
from scripts.microbench.gpu_attn_bench import timeit  # noqa: E402

b, s, h, hd = 4, 4096, 32, 64
x = [torch.randn(b, s, h, hd, device="cuda", dtype=torch.bfloat16, requires_grad=True) for _ in range(3)]
do = torch.randn(b, s, h, hd, device="cuda", dtype=torch.bfloat16)
t0 = time.time()
from vllm.vllm_flash_attn.cute.interface import flash_attn_func  # noqa: E402

out = flash_attn_func(*x)
out = out[0] if isinstance(out, tuple) else out
torch.autograd.grad(out, x, do)
torch.cuda.synchronize()
print(f"fa4 first call (compile) {time.time() - t0:.1f} s", flush=True)
flops = 4 * b * h * s * s * hd


def fa4_fwd():
    with torch.no_grad():
        return flash_attn_func(*x)


t_f = timeit(fa4_fwd)
o = flash_attn_func(*x)
o = o[0] if isinstance(o, tuple) else o
t_b = timeit(lambda: torch.autograd.grad(o, x, do, retain_graph=True))
print(f"fa4 fwd {t_f*1e3:.1f} us ({flops/t_f/1e9:.0f} TF/s)  bwd {t_b*1e3:.1f} us ({2.5*flops/t_b/1e9:.0f} TF/s)", flush=True)
q4, k4, v4 = (t.detach().transpose(1, 2).requires_grad_() for t in x)
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    t_cf = timeit(lambda: F.scaled_dot_product_attention(q4, k4, v4, scale=1 / math.sqrt(hd)))
    oc = F.scaled_dot_product_attention(q4, k4, v4, scale=1 / math.sqrt(hd))
    t_cb = timeit(lambda: torch.autograd.grad(oc, (q4, k4, v4), do.transpose(1, 2), retain_graph=True))
print(f"cudnn fwd {t_cf*1e3:.1f} us  bwd {t_cb*1e3:.1f} us", flush=True)
err = float((o.float() - oc.transpose(1, 2).float()).norm() / oc.float().norm())
print(f"fa4 vs cudnn rel err {err:.2e}")
