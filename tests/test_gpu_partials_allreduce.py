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
