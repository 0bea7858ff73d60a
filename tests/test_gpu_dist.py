"""The row-sharded solve (dist.py) on the GPU through a real NCCL process
group.  Only one B200 exists in this environment, so the group has one rank:
the allreduces are identities and the sharded path (pattern CSR of the rank's
block, sketch + allreduce, step-wise loop around the per-iteration
allreduce, `done` polling) must reproduce the single-GPU solve bit for bit.
The multi-rank host logic is covered with gloo (test_dist_gloo.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,kappa,beta,d,variant", [(20000, 60, 1e8, 1e-6, 1200, "basic"),
                                                        (50000, 200, 1e10, 1e-10, 4000, "momentum"),
                                                        (3001, 17, 1e4, 1e-3, 340, "damped")])
def test_sharded_solve_matches_single_gpu(nccl_group, m, n, kappa, beta, d, variant):
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200.dist import iterative_sketching_sharded

    p = itsk.gen_randsvd(m, n, kappa, beta, 3)
    cfg = itsk.SolverConfig(d=d, variant=variant, rng_seed=3)
    ref = itsk.iterative_sketching(p.a, p.b, cfg, p.truth, residuals="last")
    got = iterative_sketching_sharded(p.a, p.b, itsk.SolverConfig(d=d, variant=variant, rng_seed=3), m, 0, p.truth)
    assert got.trace.stop_reason == ref.trace.stop_reason
    assert got.iterations == ref.iterations
    assert np.array_equal(got.solution, ref.solution)
    assert got.trace.fe == ref.trace.fe and got.trace.re == ref.trace.re
    assert got.trace.normest == ref.trace.normest and got.trace.condest == ref.trace.condest


def test_sharded_sparse_solve_matches_single_gpu(nccl_group):
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200.dist import iterative_sketching_sharded

    p = itsk.gen_sparse(40000, 80, 2)
    cfg = itsk.SolverConfig(d=2400, max_iters=15, rng_seed=2)
    ref = itsk.iterative_sketching(p.a, p.b, cfg, residuals="last")
    got = iterative_sketching_sharded(p.a, p.b, itsk.SolverConfig(d=2400, max_iters=15, rng_seed=2), 40000, 0)
    assert got.trace.stop_reason == ref.trace.stop_reason and got.iterations == ref.iterations
    assert np.array_equal(got.solution, ref.solution)
