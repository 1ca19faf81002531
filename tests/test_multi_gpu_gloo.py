"""World-size-2 gloo tests of the multi-learner host logic on CPU: column
sharding, the partials all-reduce and max-over-ranks.  Each rank computes its
shard's partials with the CPU oracle (test infrastructure), all-reduces them,
and the sum must equal the oracle's partials of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_01561_b200 import learner


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1802_01561_b200 import workload as wl
        inp = wl.make_inputs(name, B=36)
        b0, b1 = learner.shard_columns(inp["B"], world, rank)
        sh = wl.column_slice(inp, b0, b1)
        parts = torch.from_numpy(oracle.loss_and_grad(sh, reward_mode=inp["reward_mode"])["partials"])
        learner.allreduce_partials(parts)
        t = learner.max_over_ranks(float(rank) + 0.5)
        q.put((rank, parts.numpy().copy(), t, (b0, b1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["atari", "dmlab"])
def test_partials_allreduce_equals_full_batch(name):
    import oracle
    from paper_1802_01561_b200 import workload as wl
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inp = wl.make_inputs(name, B=36)
    full = oracle.loss_and_grad(inp, reward_mode=inp["reward_mode"])["partials"]
    blocks = sorted(r[3] for r in res)
    assert blocks == [(0, 18), (18, 36)]
    for rank, parts, tmax, _ in res:
        np.testing.assert_allclose(parts, full, rtol=1e-12)
        assert tmax == 1.5


def test_shard_columns_cover():
    for B in (1, 7, 8192, 1001):
        for world in (1, 2, 3, 4, 8):
            if world > B:
                continue
            blocks = [learner.shard_columns(B, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == B
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a1 > a0
    with pytest.raises(ValueError):
        learner.shard_columns(8, 2, 2)


def test_gradient_norm():
    p = torch.tensor([0, 0, 0, 0, 9.0, 16.0, 0, 0], dtype=torch.float64)
    assert learner.gradient_norm(p) == 5.0


def _grad_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import rmsprop_oracle as ro
        from paper_1802_01561_b200 import workload as wl
        inp = wl.update_inputs(1000, seed=4, learners=world)
        g = torch.from_numpy(inp["grads"][rank].astype(np.float64))
        learner.allreduce_grads(g)  # SUM over learners (reading r11)
        theta, ms, norm = ro.rmsprop_step(inp["params"], inp["mean_square"], g.numpy(),
                                          6e-4, 0.99, 0.01, 40.0)
        q.put((rank, g.numpy().copy(), theta, ms, norm))
    finally:
        dist.destroy_process_group()


def test_gradient_allreduce_gives_identical_replicas():
    """NEXT #4 host logic: the learners' gradients are summed (NCCL on GPUs, gloo
    here) and every learner applies the same clipped RMSProp step: the replicas
    agree bitwise and equal one learner updating with the whole batch's gradient."""
    from oracle import rmsprop_oracle as ro
    from paper_1802_01561_b200 import workload as wl
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    inp = wl.update_inputs(1000, seed=4, learners=world)
    total = ro.sum_learner_grads(inp["grads"])
    theta, ms, norm = ro.rmsprop_step(inp["params"], inp["mean_square"], total, 6e-4, 0.99,
                                      0.01, 40.0)
    assert norm > 40.0  # the clip is active
    (_, g0, t0, m0, n0), (_, g1, t1, m1, n1) = res
    assert np.array_equal(g0, g1) and np.array_equal(t0, t1) and np.array_equal(m0, m1)
    np.testing.assert_allclose(g0, total, rtol=1e-15)
    np.testing.assert_allclose(t0, theta, rtol=1e-14)
    assert n0 == pytest.approx(norm, rel=1e-14)


def _oracle_kernel(*args, out, **kw):
    """LearnerStep's per-shard compute, on the CPU: the fp64 oracle on the shard's
    tensors (test infrastructure standing in for the CUDA kernel)."""
    import oracle
    from paper_1802_01561_b200 import vtrace as vt
    inp = {k: a.numpy() for k, a in zip(vt.INPUT_NAMES, args)}
    T, B, A = inp["target_logits"].shape
    inp.update(T=T, B=B, A=A, dtype=0)
    r = oracle.loss_and_grad(inp, **kw)
    out["partials"].copy_(torch.from_numpy(r["partials"]))
    out["grad_values"].copy_(torch.from_numpy(r["grad_values"]))
    out["grad_target_logits"].copy_(torch.from_numpy(r["grad_target_logits"]))


def _step_worker(rank, world, port, name, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_01561_b200 import vtrace as vt
        from paper_1802_01561_b200 import workload as wl
        full = wl.make_inputs(name, B=B, dtype=wl.DTYPE_F32)
        b0, b1 = learner.shard_columns(B, world, rank, align=4)
        sh = wl.column_slice(full, b0, b1)
        step = learner.LearnerStep(sh["T"], sh["B"], sh["A"], torch.float32, device="cpu",
                                   kernel=_oracle_kernel, reward_mode=sh["reward_mode"])
        assert step.world == world and step.rank == rank
        x = {k: torch.from_numpy(np.ascontiguousarray(sh[k])) for k in vt.INPUT_NAMES}
        out = {"grad_target_logits": torch.zeros(sh["T"], sh["B"], sh["A"], dtype=torch.float64),
               "grad_values": torch.zeros(sh["T"], sh["B"], dtype=torch.float64),
               "partials": torch.zeros(8, dtype=torch.float64)}
        step.run([(x, out)])
        q.put((rank, out["partials"].numpy().copy(), out["grad_values"].numpy().copy(), (b0, b1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_learner_step_strong_scaling(world):
    """LearnerStep (the product's multi-learner step) at world sizes 2 and 8 over gloo:
    the global batch B = 64 column-sharded in 4-column units (strong scaling, the
    BASELINE multi-GPU config), each rank's kernel (here the oracle) on its shard, the
    partials SUM-all-reduced: every rank holds the whole batch's partials and
    its shard's gradient is the matching slice of the whole batch's."""
    import oracle
    from paper_1802_01561_b200 import workload as wl
    B = 64
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, "atari", B, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = wl.make_inputs("atari", B=B, dtype=wl.DTYPE_F32)
    ref = oracle.loss_and_grad(full, reward_mode=full["reward_mode"])
    assert [r[3] for r in res] == [learner.shard_columns(B, world, r, 4) for r in range(world)]
    assert res[0][3][0] == 0 and res[-1][3][1] == B
    for rank, parts, gv, (b0, b1) in res:
        np.testing.assert_allclose(parts, ref["partials"], rtol=1e-12)
        np.testing.assert_array_equal(gv, ref["grad_values"][:, b0:b1])


def test_shard_columns_align():
    assert learner.shard_columns(8192, 8, 3, align=8) == (3072, 4096)
    assert learner.shard_columns(40, 3, 0, align=8) == (0, 16)
    assert learner.shard_columns(40, 3, 2, align=8) == (32, 40)
    with pytest.raises(ValueError):
        learner.shard_columns(30, 2, 0, align=8)
