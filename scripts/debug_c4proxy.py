import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200 import solvers
from oracle import itsketch_oracle as orc
m, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a,b,t = orc.gen_randsvd(m,n,1e8,1e-6,0)
p = orc.sparse_sign_pattern(d,m,8,0)
sab = orc.sketch_apply(p, np.column_stack([a, b]))
s = itsk.sparse_sign_new(d, m, 8, 0)
w = s.apply_dense(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
print("sketch bitwise:", np.array_equal(w.cpu().numpy(), sab))
q, r = orc.householder_qr_econ(sab[:, :n])
R, z = itsk.linalg.qr_aug(w, n)
Rn = R.cpu().numpy()
print("R rel err", np.linalg.norm(Rn - r)/np.linalg.norm(r))
err = np.abs(Rn - r)
i, j = np.unravel_index(np.argmax(err), err.shape)
print("max err at", i, j, err[i,j], r[i,j])
rowerr = np.linalg.norm(Rn - r, axis=1)/np.linalg.norm(r, axis=1)
print("rows with err>1e-10:", np.nonzero(rowerr > 1e-10)[0][:40])
print("z err", np.linalg.norm(z.cpu().numpy() - q.T@sab[:, n]) / np.linalg.norm(q.T@sab[:,n]))
