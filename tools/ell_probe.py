"""ELL vs CSR SpMV on B200 (kernel-level, CUDA events, 50 back-to-back
launches each; inputs: C2 matrix 1024^2 (5 nnz/row) and random rows (9/row,
n = 2M)).  Algorithmic bytes: CSR 12 nnz + 4 (n+1) + 16 n; ELL 12 n width + 16 n."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200 import fused  # noqa: E402


def t(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


out = {}
for name, (a, _) in (("convdiff2d_1024", pk.convdiff2d(1024)), ("random_2M_9", pk.gen_random_rowwise(2 << 20, 9, 1))):
    e = pk.csr_to_ell(a)
    x = torch.rand(a.n_cols, dtype=torch.float64, device="cuda")
    n, nnz = a.n_rows, a.nnz
    us_csr = t(lambda: fused.spmv(a, x))
    us_ell = t(lambda: pk.spmv_ell(e, x))
    out[name] = {"n": n, "nnz": nnz, "width": e.width,
                 "csr_us": round(us_csr, 2), "csr_gbs": round((12 * nnz + 4 * (n + 1) + 16 * n) / us_csr / 1e3, 1),
                 "ell_us": round(us_ell, 2), "ell_gbs": round((12 * n * e.width + 16 * n) / us_ell / 1e3, 1)}
print(json.dumps(out))
