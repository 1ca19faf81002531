"""Row a13 over NVLink peer memory (vtrace_partials_allreduce): the learners'
partials summed in learner order, bitwise identical on every learner.  On one GPU the
learners are simulated by concurrent kernels on separate streams with their mailboxes
in the same device memory (the protocol is the same; peer mapping is what NVLink adds)."""
import pytest
import torch

from paper_1802_01561_b200 import vtrace as vt


def _run(n, calls, inplace, seed):
    dev = torch.device("cuda", 0)
    nb = vt.partials_mailbox_bytes(n)
    assert nb == 2 * n * 8 * 16
    mbs = [torch.zeros(nb // 8, dtype=torch.float64, device=dev) for _ in range(n)]
    ptrs = [m.data_ptr() for m in mbs]
    counters = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(n)]
    streams = [torch.cuda.Stream(dev) for _ in range(n)]
    g = torch.Generator().manual_seed(seed)
    for call in range(calls):
        parts = [(torch.randn(8, dtype=torch.float64, generator=g) * 10 ** (r % 3)).to(dev)
                 for r in range(n)]
        host = [p.cpu() for p in parts]
        outs = [p if inplace else torch.full((8,), -1.0, dtype=torch.float64, device=dev)
                for p in parts]
        torch.cuda.synchronize()
        for r in reversed(range(n)):  # the last learner first: the others wait for it
            with torch.cuda.stream(streams[r]):
                vt.partials_allreduce(parts[r], ptrs, r, counters[r], out=outs[r])
        torch.cuda.synchronize()
        expect = torch.zeros(8, dtype=torch.float64)
        for r in range(n):  # the kernel's order: 0 + p_0 + p_1 + ...
            expect = expect + host[r]
        for r in range(n):
            assert torch.equal(outs[r].cpu(), expect), (call, r)
    for c in counters:
        assert int(c.item()) == calls


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_partials_allreduce_learners_on_one_gpu(n):
    _run(n, calls=5, inplace=False, seed=n)


@pytest.mark.gpu
def test_partials_allreduce_in_place_many_calls():
    """Both mailbox parities, many calls in a row, output over the input."""
    _run(2, calls=40, inplace=True, seed=11)


@pytest.mark.gpu
def test_learners_sum_inside_the_vtrace_kernel_with_simulated_peer():
    """vtrace_loss_and_grad_learners on one GPU, learner 0 of 2: the peer is simulated by its
    slots in learner 0's mailbox, written before each call with the call's tag (the
    workspace's call count + 1).  The kernel's partials must be (own, bitwise as the plain
    call) + (peer) in learner order, the gradients unchanged, and learner 0's own slot must
    land in the peer's mailbox."""
    import paper_1802_01561_b200 as pkg
    from paper_1802_01561_b200 import workload as wl
    inp = wl.make_inputs("large", T=24, B=512)
    T, B, A = inp["T"], inp["B"], inp["A"]
    assert pkg.kernel_for(T, B, A, inp["dtype"]).startswith("vtrace_cb_kernel")
    d = pkg.tensors_from_workload(inp, "cuda")
    args = [d[k] for k in vt.INPUT_NAMES]
    ws_plain = pkg.Workspace(T, B, A, inp["dtype"])
    ws = pkg.Workspace(T, B, A, inp["dtype"])
    nb = vt.partials_mailbox_bytes(2)
    mb = [torch.zeros(nb // 8, dtype=torch.float64, device="cuda") for _ in range(2)]
    g = torch.Generator().manual_seed(3)
    for call in range(4):
        plain = pkg.loss_and_grad(*args, workspace=ws_plain, reward_mode=inp["reward_mode"])
        peer = torch.randn(8, dtype=torch.float64, generator=g) * 100
        tag = call + 1
        base = ((tag & 1) * 2 + 1) * 8  # slots [parity][learner 1][k]
        for k in range(8):
            mb[0][2 * (base + k)] = float(peer[k])
            mb[0].view(torch.int64)[2 * (base + k) + 1] = tag
        out = pkg.loss_and_grad(*args, workspace=ws, reward_mode=inp["reward_mode"],
                                mailboxes=[m.data_ptr() for m in mb], self_index=0)
        torch.cuda.synchronize()
        own = plain["partials"].cpu()
        assert torch.equal(out["partials"].cpu(), (0.0 + own) + peer)
        assert torch.equal(out["grad_target_logits"], plain["grad_target_logits"])
        assert torch.equal(out["grad_values"], plain["grad_values"])
        mine = ((tag & 1) * 2 + 0) * 8  # learner 0's slots in the peer's mailbox
        got = torch.tensor([float(mb[1][2 * (mine + k)]) for k in range(8)], dtype=torch.float64)
        assert torch.equal(got, own)


@pytest.mark.gpu
@pytest.mark.parametrize("n,batches", [(2, [8, 8, 3]), (4, [1, 32, 5])])
def test_partials_allreduce_batched(n, batches):
    """vtrace_partials_allreduce_batched: several steps' partials summed over the learners
    in one kernel, in place, learner order, bitwise identical on every learner; batch sizes
    vary from call to call (every learner the same) within the mailbox's maximum."""
    dev = torch.device("cuda", 0)
    bmax = max(batches)
    nb = vt.partials_mailbox_bytes_batched(n, bmax)
    assert nb == 2 * n * bmax * 8 * 16
    mbs = [torch.zeros(nb // 8, dtype=torch.float64, device=dev) for _ in range(n)]
    ptrs = [m.data_ptr() for m in mbs]
    counters = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(n)]
    streams = [torch.cuda.Stream(dev) for _ in range(n)]
    g = torch.Generator().manual_seed(7 + n)
    for call, m in enumerate(batches):
        parts = [[(torch.randn(8, dtype=torch.float64, generator=g) * 10 ** (r % 3)).to(dev)
                  for _ in range(m)] for r in range(n)]
        host = [[p.cpu() for p in pr] for pr in parts]
        torch.cuda.synchronize()
        for r in reversed(range(n)):
            with torch.cuda.stream(streams[r]):
                vt.partials_allreduce_batched(parts[r], ptrs, r, counters[r], batch_max=bmax)
        torch.cuda.synchronize()
        for s in range(m):
            expect = torch.zeros(8, dtype=torch.float64)
            for r in range(n):
                expect = expect + host[r][s]
            for r in range(n):
                assert torch.equal(parts[r][s].cpu(), expect), (call, s, r)
    for c in counters:
        assert int(c.item()) == len(batches)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_partials_allreduce_batched_back_to_back(n):
    """Batched calls of different sizes queued back to back on every learner's stream (no
    host synchronisation between calls, so one learner can run a call ahead of another): the
    mailbox regions of the two parities must not overlap whatever the batch sizes."""
    dev = torch.device("cuda", 0)
    sizes = [8, 1, 5, 8, 3, 8, 2, 7, 8, 1]
    bmax = 8
    mbs = [torch.zeros(vt.partials_mailbox_bytes_batched(n, bmax) // 8, dtype=torch.float64,
                       device=dev) for _ in range(n)]
    ptrs = [m.data_ptr() for m in mbs]
    counters = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(n)]
    streams = [torch.cuda.Stream(dev) for _ in range(n)]
    g = torch.Generator().manual_seed(40 + n)
    calls = [[[(torch.randn(8, dtype=torch.float64, generator=g)).to(dev) for _ in range(m)]
              for r in range(n)] for m in sizes]
    expect = [[sum((c[r][s].cpu() for r in range(n)), torch.zeros(8, dtype=torch.float64))
               for s in range(len(c[0]))] for c in calls]
    torch.cuda.synchronize()
    for r in reversed(range(n)):
        with torch.cuda.stream(streams[r]):
            for c in calls:
                vt.partials_allreduce_batched(c[r], ptrs, r, counters[r], batch_max=bmax)
    torch.cuda.synchronize()
    for i, c in enumerate(calls):
        for s in range(len(c[0])):
            for r in range(n):
                assert torch.equal(c[r][s].cpu(), expect[i][s]), (i, s, r)
