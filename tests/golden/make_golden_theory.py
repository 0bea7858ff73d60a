"""Golden values for the convergence-theory yardsticks the acceptance tests
use (tests/test_gpu_acceptance.py): the reference's rate functions and bound
curves (solvers.py:102-171) and measure_distortion (embed.py:118-130) on the
exact inputs of its acceptance criteria C02 / C08 and test_solvers.py's
geometric-contraction and theorem-surrogate tests.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_theory.py

Imports the UNMODIFIED reference from /root/reference/pkg/src (or
$ITSKETCH_REF); writes tests/golden/theory.npz.
"""
import os
import sys

import numpy as np

REF = os.environ.get("ITSKETCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from itsketch.embed import measure_distortion, sparse_sign_new  # noqa: E402
from itsketch.problems import gen_randsvd  # noqa: E402
from itsketch.solvers import rate_g_damp, rate_g_is, rate_g_mom, theoretical_bound_curve  # noqa: E402

out = {}
eps_grid = np.array([0.0, 0.05, 0.1, 0.2, 0.2236, 0.25, 0.28])
out["eps_grid"] = eps_grid
out["rate_is"] = np.array([rate_g_is(e) for e in eps_grid])
out["rate_damp"] = np.array([rate_g_damp(e) for e in eps_grid])
out["rate_mom"] = np.array([rate_g_mom(e) for e in eps_grid])
for v, first in (("basic", 0), ("damped", 0), ("momentum", 2)):
    fe, re = theoretical_bound_curve(v, 0.2, 1e4, 1.5, 1e-3, 12, first_iter=first)
    out[f"bound_{v}_fe"], out[f"bound_{v}_re"] = fe, re
# distortion of the embeddings the acceptance tests measure
cases = {
    "c02": ((2000, 50, 1e2, 1e-3, 0), (1000, 2000, 8, 1), True),
    "geo": ((1000, 20, 10.0, 1e-3, 1), (400, 1000, 8, 1), False),
    "thm": ((1000, 20, 100.0, 1e-3, 2), (400, 1000, 8, 2), False),
}
for name, (prob, emb, with_b) in cases.items():
    p = gen_randsvd(*prob)
    s = sparse_sign_new(*emb)
    basis = np.linalg.qr(np.column_stack([p.a, p.b]) if with_b else p.a, mode="reduced")[0]
    out[f"eps_{name}"] = np.array(measure_distortion(s, basis).epsilon)
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "theory.npz"), **out)
print({k: (v.tolist() if v.size < 8 else v.shape) for k, v in out.items()})
