import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle
from paper_2511_18207_b200 import Context, option
ctx = Context(0)
for D in (128, 136, 160, 176, 192):
    rng = np.random.default_rng(D + 5)
    A = (rng.standard_normal((700, D)) * 1e-6).astype(np.float32)
    B = (rng.standard_normal((900, D)) * 1e-6 + 2e-7).astype(np.float32)
    A[3], A[4] = 1e4, -1e4
    B[5], B[600] = -1e4, 1e4
    ref, arg = oracle.row_minima(A, B)
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    rm = ctx.directed_hd_rowmin(At, Bt).cpu().numpy()
    bad = np.abs(rm - ref) > 1e-5 * (ref + 1e-12)
    print(D, "bad rows", int(bad.sum()), "first", np.nonzero(bad)[0][:6], rm[bad][:4], ref[bad][:4], flush=True)
    # scale sweep: multiply the whole problem by 2^s
    for s in (8, 16):
        rm2 = ctx.directed_hd_rowmin(At * 2.0 ** s, Bt * 2.0 ** s).cpu().numpy() / 4.0 ** s
        print("   x2^%d bad rows" % s, int((np.abs(rm2 - ref) > 1e-5 * (ref + 1e-12)).sum()), flush=True)
    A2, B2 = A.copy(), B.copy()
    A2[3], A2[4], B2[5], B2[600] = 1e2, -1e2, -1e2, 1e2
    ref2, _ = oracle.row_minima(A2, B2)
    rm3 = ctx.directed_hd_rowmin(torch.from_numpy(A2).cuda(), torch.from_numpy(B2).cuda()).cpu().numpy()
    print("   outliers 1e2: bad rows", int((np.abs(rm3 - ref2) > 1e-5 * (ref2 + 1e-12)).sum()), flush=True)
