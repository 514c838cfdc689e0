import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import datagen, oracle
from paper_1906_06496_b200 import tem
from test_gpu_parity import oracle_with_gpu_decisions
N, B, lam, lr = 2, 2, (2.0, 1.0, 1.0), 0.05
p = datagen.init_params()
sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, precision=0, lr=lr, loss_weight=lam)
s = tem.TemSession(sc, p)
x = np.stack([datagen.features(B, rank=r) for r in range(N)])
lab = np.stack([datagen.labels(B, rank=r) for r in range(N)])
s.step(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda())
print("sync", s.sync())
for r in range(N):
    g = s.local_grad(r).cpu().numpy()[:s.K]
    ref = oracle.tem_fwd_bwd(x[r], p, lab[r], lam, prec=0)
    d = np.abs(g - ref["grad"]); i = int(d.argmax())
    print(r, "err", d.max() / np.abs(ref["grad"]).max(), "at", i, g[i], ref["grad"][i])
    ref2 = oracle_with_gpu_decisions(oracle, s, r, x[r], p, lab[r], lam, 0)
    print(r, "err with gpu decisions", np.abs(g - ref2["grad"]).max() / np.abs(ref2["grad"]).max())
    z = s.logits(r).cpu().numpy(); print("z err", np.abs(z - ref["z"].reshape(z.shape)).max())
print("path", s.kernel_path())
