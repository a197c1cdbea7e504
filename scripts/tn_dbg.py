import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2006_06608_b200.capi import Context
from paper_2006_06608_b200.gcn import ctx_gemm_tn
ctx = Context(0)
for (m, p, q) in ((32, 32, 32), (8, 32, 32), (32, 4, 4), (64, 96, 16)):
    rng = np.random.default_rng(1)
    a = rng.integers(-3, 4, (m, p)).astype(np.float32)
    b = rng.integers(-3, 4, (m, q)).astype(np.float32)
    got = ctx_gemm_tn(ctx, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    want = a.T @ b
    print((m, p, q), "ok" if np.array_equal(got, want) else "BAD", "nnz got", int((got != 0).sum()), "of", got.size)
    if not np.array_equal(got, want):
        print(" got[:4,:8]\n", got[:4, :8], "\n want[:4,:8]\n", want[:4, :8])
        # candidate: rows of got permuted?
        for i in range(min(4, p)):
            hits = [k for k in range(p) if np.array_equal(got[i], want[k])]
            print("  got row", i, "matches want rows", hits)
