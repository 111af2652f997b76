"""Multi-rank (subdomain-sharded) Algorithm 1: the host protocol of
paper_2509_23180_b200/dist.py run with world_size 2 and 3 over gloo on CPU,
with the oracle as the local arithmetic, against the single-process oracle
solve.  (On GPUs the same code runs over NCCL with the native backend.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fftddm_oracle as O
from paper_2509_23180_b200 import configs, dist as pdist, krylov


class OracleBackend:
    def plan(self, sub):
        return O.plan(sub)

    def solve(self, pl, v):
        return O.solve(pl, np.asarray(v, dtype=float))

    def array(self, x):
        return np.array(x, dtype=float).reshape(-1)

    def zeros(self, n):
        return np.zeros(n)

    def index(self, idx):
        return np.asarray(idx)

    def comm(self, x):
        return torch.from_numpy(np.ascontiguousarray(x, dtype=float))

    def empty_comm(self, n):
        return torch.empty(n, dtype=torch.float64)

    def from_comm(self, t):
        return t.numpy()

    def gmres(self, op, rhs, cfg):
        return O.gmres(op, rhs, m=cfg.m, tol=cfg.tol, max_restarts=cfg.max_restarts)

    def norm(self, v):
        return float(np.linalg.norm(v))

    def stencil(self, sub, v):
        return O.apply_operator(sub, v)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, kappa, outdir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        comp = configs.cross_composite(N, kappa=kappa)
        f, _ = configs.manufactured_rhs(comp, "sin_exp")
        fields, rep = pdist.dist_ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10),
                                           backend=OracleBackend())
        np.savez(os.path.join(outdir, f"rank{rank}.npz"),
                 **{f"f{sid}": np.asarray(v) for sid, v in fields.items()},
                 iters=np.array(rep.iterations if rep else -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("N,kappa", [(8, 0.0), (15, -100.0)])
def test_sharded_solve_matches_single_process_ws(tmp_path, world, N, kappa):
    _run_and_compare(tmp_path, world, N, kappa)


def test_more_ranks_than_arms(tmp_path):
    """world 6 > 4 arms + 1: the rank without an arm returns at once instead of
    waiting for commands that never come."""
    _run_and_compare(tmp_path, 6, 8, 0.0)


def _fail_worker(rank, world, port, outdir):
    from paper_2509_23180_b200.errors import ConvergenceError
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        comp = configs.cross_composite(15, kappa=0.0)
        f, _ = configs.manufactured_rhs(comp, "sin_exp")
        be = OracleBackend()
        if rank == 0:
            def gmres(op, rhs, cfg):
                raise ConvergenceError("forced")
            be.gmres = gmres
        status = "ok"
        try:
            pdist.dist_ddm_solve(comp, f, krylov.GmresConfig(m=50, tol=1e-10), backend=be)
        except ConvergenceError:
            status = "raised"
        with open(os.path.join(outdir, f"rank{rank}.txt"), "w") as fh:
            fh.write(status)
    finally:
        dist.destroy_process_group()


def test_gmres_failure_releases_workers(tmp_path):
    """GMRES raising on rank 0 still sends CMD_DONE: the arm ranks return."""
    port = _free_port()
    mp.spawn(_fail_worker, args=(3, port, str(tmp_path)), nprocs=3, join=True)
    assert (tmp_path / "rank0.txt").read_text() == "raised"
    assert (tmp_path / "rank1.txt").read_text() == "ok"
    assert (tmp_path / "rank2.txt").read_text() == "ok"


def _run_and_compare(tmp_path, world, N, kappa):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, N, kappa, str(tmp_path)), nprocs=world, join=True)
    comp = configs.cross_composite(N, kappa=kappa)
    f, _ = configs.manufactured_rhs(comp, "sin_exp")
    ref, rep = O.ddm_solve(comp, f, m=50, tol=1e-10)
    got, iters = {}, None
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        for k in d.files:
            if k.startswith("f"):
                got[int(k[1:])] = d[k]
        if r == 0:
            iters = int(d["iters"])
    assert sorted(got) == sorted(ref)
    assert iters == rep.iterations
    for sid in ref:
        np.testing.assert_allclose(got[sid], ref[sid], rtol=0, atol=1e-12 * np.abs(ref[sid]).max())


def test_owner_assignment():
    assert pdist.owners(4, 1) == [0, 0, 0, 0]
    assert pdist.owners(4, 2) == [1, 1, 1, 1]
    assert pdist.owners(4, 3) == [1, 2, 1, 2]
    assert pdist.owners(4, 5) == [1, 2, 3, 4]
