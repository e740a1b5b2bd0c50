"""Dev: sharded int8 moments (prohd_local_colmax -> MAX -> prohd_local_moments_i8) vs the one-shot
covariance and the fp64 two-pass covariance, per shard count."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import datagen
from oracle import prohd as OP
from paper_2511_18207_b200 import Context
from paper_2511_18207_b200.dist import CudaPhases, row_range
ctx = Context(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
A, B = datagen.generate(cfg, n=n)
At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
D = A.shape[1]
rmu, rC = OP.covariance(A, B)
mu1, C1, path = ctx.covariance(At, Bt)
print("one-shot path", path, "max|dC|", np.abs(C1 - rC).max(), "max|C|", np.abs(rC).max())
ph = CudaPhases(ctx, dmma=False)
s = ph.shift(At[:4096], Bt[:4096])
print("shift max", np.abs(s).max())
N = A.shape[0] + B.shape[0]
for G in (1, 2, 4):
    la = [row_range(A.shape[0], g, G) for g in range(G)]
    lb = [row_range(B.shape[0], g, G) for g in range(G)]
    cms = [ph.local_colmax(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s) for g in range(G)]
    cm = cms[0]
    for c in cms[1:]:
        cm = torch.maximum(cm, c)
    for dm in (False, True):
        mom = sum((ph.ctx.local_moments_i8(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s, cm) if not dm else
                   ph.ctx.local_moments(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s)) for g in range(G))
        m = mom.cpu().numpy()
        SA, SB, Gm = m[:D], m[D:2 * D], m[2 * D:].reshape(D, D)
        mu = (SA + SB) / N
        C = Gm / N - np.outer(mu, mu)
        d = np.abs(C - rC)
        i, j = np.unravel_index(d.argmax(), d.shape)
        print(f"G={G} {'dmma' if dm else 'i8  '}: max|dC| {d.max():.3e} at ({i},{j}) C={C[i, j]:.6e} ref={rC[i, j]:.6e}; "
              f"max|dS_A| {np.abs(SA - (A.astype(np.float64) - s).sum(0)).max():.3e}", flush=True)
# directions from the last sharded moments of each kind vs numpy eigh of the same C
k = datagen.CONFIGS[cfg].k
for dm in (False, True):
    G = 4
    la = [row_range(A.shape[0], g, G) for g in range(G)]
    lb = [row_range(B.shape[0], g, G) for g in range(G)]
    mom = sum((ph.ctx.local_moments_i8(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s, cm) if not dm else
               ph.ctx.local_moments(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s)) for g in range(G))
    dirs, nd = ph.directions(mom, A.shape[0], B.shape[0], D, k, s)
    U = dirs.cpu().numpy()
    m = mom.cpu().numpy()
    mu = (m[:D] + m[D:2 * D]) / N
    C = m[2 * D:].reshape(D, D) / N - np.outer(mu, mu)
    w, V = np.linalg.eigh(C)
    top = V[:, ::-1][:, :k]
    ang = [abs(abs(U[1 + i] @ top[:, i]) - 1) for i in range(k)]
    print(("dmma" if dm else "i8  "), "nd", nd, "top lam", w[::-1][:4], "max 1-|cos|", max(ang), "U[1][:4]", U[1][:4],
          "sym", np.abs(C - C.T).max(), flush=True)
    print("   mom finite", np.isfinite(m).all(), "G diag min", np.diag(m[2 * D:].reshape(D, D)).min())
# the int8 sharded moments, G symmetrised on the host
G = 4
mom = sum(ph.ctx.local_moments_i8(At[la[g][0]:la[g][1]], Bt[lb[g][0]:lb[g][1]], s, cm) for g in range(G))
m = mom.cpu().numpy().copy()
Gm = m[2 * D:].reshape(D, D)
for name, Gx in (("asym", Gm), ("sym", 0.5 * (Gm + Gm.T)), ("asymT", Gm.T.copy())):
    mm = np.concatenate([m[:2 * D], Gx.ravel()])
    dirs, nd = ph.directions(torch.from_numpy(mm).cuda(), A.shape[0], B.shape[0], D, k, s)
    U = dirs.cpu().numpy()
    print(name, "U[1][:3]", U[1][:3], "U[2][:3]", U[2][:3], flush=True)
