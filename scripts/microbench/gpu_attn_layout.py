"""cuDNN SDPA fwd+bwd at the CoLA-1B step shape (b4 h32 s4096 hd64): BSHD-strided views (what the
executor passes) vs BHSD-contiguous inputs (run on the box; not a pytest module)."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

b, h, s, hd = 4, 32, 4096, 64
dev, bf = "cuda", torch.bfloat16


def run(q, k, v, do, reps=10):
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        for _ in range(3):
            o = F.scaled_dot_product_attention(q, k, v)
            torch.autograd.grad(o, (q, k, v), do)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        tf = tb = 0.0
        for _ in range(reps):
            e0.record()
            o = F.scaled_dot_product_attention(q, k, v)
            e1.record()
            torch.autograd.grad(o, (q, k, v), do)
            e2.record()
            torch.cuda.synchronize()
            tf += e0.elapsed_time(e1)
            tb += e1.elapsed_time(e2)
    return tf / reps * 1e3, tb / reps * 1e3


x = torch.randn(3, b * s, h * hd, device=dev, dtype=bf)
bshd = [x[i].view(b, s, h, hd).transpose(1, 2).detach().requires_grad_() for i in range(3)]
do_s = torch.randn(b * s, h * hd, device=dev, dtype=bf).view(b, s, h, hd).transpose(1, 2)
print("BSHD strided:   fwd %.1f us  bwd %.1f us" % run(*bshd, do_s))
bhsd = [t.detach().contiguous().requires_grad_() for t in bshd]
print("BHSD contiguous: fwd %.1f us  bwd %.1f us" % run(*bhsd, do_s.contiguous()))
