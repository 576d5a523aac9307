"""Multi-GPU subtree partition, tested on CPU: partition
invariants on the BASELINE trees and the point-to-point update exchange with
the gloo backend at world size 2 (127.0.0.1 rendezvous)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1502_07405_b200 as P
from paper_1502_07405_b200.parallel import exchange_updates, subtree_partition


@pytest.mark.parametrize("kind,k,leaf,nranks", [("p3d", 32, 32, 2), ("p3d", 32, 32, 8),
                                                  ("p2d", 64, 16, 4), ("p3d", 48, 32, 8)])
def test_partition_invariants(kind, k, leaf, nranks):
    op = P.ordered_grid(kind, k, leaf)
    t = op.t
    part = subtree_partition(t, nranks)
    # every front owned, every rank owns one contiguous subtree + top fronts
    assert (part.owner >= 0).all() and (part.owner < nranks).all()
    for r, s in enumerate(part.roots):
        ids = part.fronts_of(r)
        sub = ids[ids <= s]
        assert sub.max() == s and np.all(np.diff(sub) == 1)  # contiguous postorder range
    # separators of a rank's subtree are a contiguous index range
    for r, s in enumerate(part.roots):
        ids = [i for i in part.fronts_of(r) if i <= s]
        lo, hi = t.sep_begin[min(ids)], t.sep_end[s]
        assert sum(t.sep_end[i] - t.sep_begin[i] for i in ids) == hi - lo
    # exchanges only along tree edges that cross ranks, exactly 2^L - 1 of them
    assert len(part.edges) == nranks - 1
    for (c, p, src, dst, nu) in part.edges:
        assert t.parent[c] == p and src != dst and part.owner[c] == src and part.owner[p] == dst
    # the partition does not change the integer structure (upd sets, levels)
    op2 = P.ordered_grid(kind, k, leaf)
    assert np.array_equal(op2.t.upd_ind, t.upd_ind)


def test_partition_c5_top_levels():
    op = P.ordered_grid("p3d", 128, 32)
    part = subtree_partition(op.t, 8)
    assert part.level == 3 and len(part.roots) == 8
    # 7 top fronts, owned by their child0 subtree's rank
    top = np.nonzero(op.t.level < 3)[0]
    assert len(top) == 7
    # the update operators crossing NVLink: nu^2 doubles per edge
    assert part.factor_bytes() > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, k, leaf, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op = P.ordered_grid(kind, k, leaf)
    part = subtree_partition(op.t, world)

    def payload(c):  # deterministic stand-in for the child's update operator
        nu = int(op.t.upd_ptr[c + 1] - op.t.upd_ptr[c])
        g = np.random.default_rng(c).standard_normal((nu, nu))
        return torch.from_numpy(g)

    def send(a, dst):
        dist.send(a.contiguous(), dst)

    def recv(shape, src):
        buf = torch.empty(shape, dtype=torch.float64)
        dist.recv(buf, src)
        return buf

    got = exchange_updates(part, rank, payload, send, recv)
    ok = all(torch.equal(v, payload(c)) for c, v in got.items())
    q.put((rank, ok, sorted(got)))
    dist.barrier()
    dist.destroy_process_group()


def test_update_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, "p3d", 24, 32, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    res.sort()
    assert all(ok for _, ok, _ in res)
    # rank 0 owns the root (child0 subtree) and receives rank 1's subtree-root update
    assert res[0][2] and not res[1][2]


# ---- the phased factor / solve protocol, with a recording stand-in engine ----
from paper_1502_07405_b200.parallel import ProtocolEngine as FakeEngine  # noqa: E402
from paper_1502_07405_b200.parallel import protocol_expected as _expected  # noqa: E402


def _phased_worker(rank, world, port, q):
    from paper_1502_07405_b200.parallel import TorchTransport, phased_factor, phased_solve
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op = P.ordered_grid("p3d", 24, 32)
    t = op.t
    part = subtree_partition(t, world)
    eng = FakeEngine(t, part, rank)
    nlev = int(t.level.max()) + 1
    tr = TorchTransport(None)
    phased_factor(part, t.level, nlev, {rank: eng}, tr)
    x = torch.zeros((1, len(t.child0)), dtype=torch.float64)
    # upd_of(c) -> nu_c copies of the parent's slot in this stand-in x
    def upd_of(c):
        return torch.full((int(t.upd_ptr[c + 1] - t.upd_ptr[c]),), int(t.parent[c]),
                          dtype=torch.long)
    phased_solve(part, t.level, nlev, upd_of, {rank: eng}, {rank: x}, 1, tr)
    val, xe = _expected(t)
    own = np.nonzero(eng.own)[0]
    ok_val = all(abs(eng.val[f] - val[f]) < 1e-9 for f in own)
    ok_x = all(abs(float(x[0, f]) - xe[f]) < 1e-9 for f in own)
    q.put((rank, ok_val, ok_x))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_phased_protocol_gloo(world):
    # every rank's phases find their children's updates / bupd and their
    # parents' x where the sequential schedule would have them
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_phased_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(ok_v and ok_x for _, ok_v, ok_x in res), res


def test_bench_spawns_ranks_dry_run():
    # `python bench.py --gpus 4` outside torchrun launches 4 ranks itself; the
    # CPU dry run (gloo) runs the phased protocol on the workload's partition
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4",
                          "--dry-run", "--config", "c3"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 4 and line["protocol_ok"] is True
    assert line["config"]["parallelism"] == "subtree4" and line["partition"]["edges"] == 3


@pytest.mark.parametrize("kind,k,leaf,nranks", [("p3d", 32, 32, 2), ("p3d", 48, 32, 8),
                                                  ("p2d", 64, 16, 4)])
def test_native_partition_matches_python(kind, k, leaf, nranks):
    # the C++ driver (csrc/mgpu.cu) partitions exactly like parallel.py
    from paper_1502_07405_b200.parallel import native_partition
    op = P.ordered_grid(kind, k, leaf)
    part = subtree_partition(op.t, nranks)
    owner, ne = native_partition(op.t, nranks)
    assert np.array_equal(owner, part.owner) and ne == len(part.edges)
