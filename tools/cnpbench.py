"""CNP stack timing at Llama-1B size (3,696 blocks of 256): fused one-kernel
forward/backward (csrc/cnp_fused.cu) vs the unfused tensor-core path
(csrc/cnp_tc.cu).  CUDA events, best of 10, inputs resident."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_05500_b200 import _native as N  # noqa: E402

nb, b = int(sys.argv[1]) if len(sys.argv) > 1 else 3696, int(sys.argv[2]) if len(sys.argv) > 2 else 256
pairs = b * (b - 1) // 2
pk = torch.randn((nb, pairs), device="cuda") * 0.01
dg = torch.randn((nb, b, b), device="cuda")
g16 = torch.empty((nb, b, b), dtype=torch.bfloat16, device="cuda")
qq2 = torch.empty((nb, b, 2 * b), dtype=torch.bfloat16, device="cuda")
gp = torch.empty_like(pk)
ws, wsb = N.workspace(N.lib().poetx_cnp_tc_workspace_bytes(nb, b))
st = N.stream_ptr()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, a.elapsed_time(e))
    return best


fwd_f = t(lambda: N.call("poetx_cnp_forward_fused", nb, b, pk.data_ptr(), g16.data_ptr(), None, st))
bwd_f = t(lambda: N.call("poetx_cnp_backward_fused", nb, b, pk.data_ptr(), dg.data_ptr(), gp.data_ptr(), 0, st))
fwd_u = t(lambda: N.call("poetx_cnp_forward_tc", nb, b, pk.data_ptr(), qq2.data_ptr(), g16.data_ptr(), None, ws, wsb, st))
bwd_u = t(lambda: N.call("poetx_cnp_backward_tc", nb, b, qq2.data_ptr(), dg.data_ptr(), gp.data_ptr(), 0, ws, wsb, st))
fl = 2.0 * b ** 3 * nb
print(f"nb={nb} b={b}")
print(f"fused   fwd {fwd_f:.3f} ms ({2 * fl / fwd_f / 1e9:.0f} TF/s on 2 products)  "
      f"bwd {bwd_f:.3f} ms ({7 * fl / bwd_f / 1e9:.0f} TF/s on 7 products)")
print(f"unfused fwd {fwd_u:.3f} ms  bwd {bwd_u:.3f} ms")
