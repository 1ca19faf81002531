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
