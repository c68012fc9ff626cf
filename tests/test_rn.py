"""GPU parity for the r_n scalability family (SURVEY.md
s8(f) NEXT-2): r_n = ([0-4]{n}[5-9]{n})* on accepted texts, and
r_a = r_n|a* on a repetition of "a".  The D-SFA grows as |D|^2 (10,100 states
at n = 50, 64,770 at n = 127, the largest that fits u16 ids), which moves the
table from bank-private shared memory to HOT rows + L2 and, for these single-
loop automata, to the FACTORED step.  Bit-exact (final state, accept) against
the oracle's Alg. 2, for the SFA path and the Alg. 3 baseline.
"""
import numpy as np
import pytest

import oracle as O
import paper_1405_0562_b200 as P
import workloads as W

pytestmark = pytest.mark.gpu

DIGITS = b"0123456789"


@pytest.fixture(scope="module")
def torch_cuda(cuda_ok):
    import torch
    return torch


def _res(torch):
    return torch.zeros(2, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("n", [10, 50, 100, 127])
def test_rn_accepted_and_perturbed(torch_cuda, n):
    torch = torch_cuda
    rx = W.rn_regex(n)
    sfa = P.SFA(rx, DIGITS)
    d = O.OracleDFA(rx, DIGITS)
    t = W.rn_accepted(n, 24 << 20)
    rng = np.random.default_rng(n)
    cases = [t, t[: t.size - 2 * n - 1]]            # accepted; a ragged prefix (rejected unless aligned)
    bad = t.copy()
    bad[int(rng.integers(0, t.size))] ^= 0x07        # one digit moved (maybe to the other half)
    cases.append(bad)
    cases.append(t[: int(rng.integers(1, 1 << 20))])
    for c in cases:
        dt = torch.from_numpy(c.copy()).cuda()
        exp = d.run(c)
        assert sfa.match(dt) == exp, (n, c.size)
        r = _res(torch)
        sfa.match_speculative(dt, r)
        torch.cuda.synchronize()
        assert tuple(int(x) for x in r.cpu().numpy().view(np.uint32)) == (exp[0], int(exp[1]))
    assert d.run(t) == (0, True)


@pytest.mark.parametrize("mode", [3, 4])  # HOT_L2, L2
def test_r50_forced_residency(torch_cuda, mode):
    torch = torch_cuda
    rx = W.rn_regex(50)
    sfa = P.SFA(rx, DIGITS)
    sfa.set_residency(mode)
    d = O.OracleDFA(rx, DIGITS)
    t = W.rn_accepted(50, 9 << 20)
    for n in (t.size, t.size - 77, 4_000_001):
        assert sfa.match(torch.from_numpy(t[:n].copy()).cuda()) == d.run(t[:n])


@pytest.mark.parametrize("n", [50, 127])
def test_ra_single_hot_state(torch_cuda, n):
    """r_a on "a"^m: every chunk stays in one SFA state."""
    torch = torch_cuda
    rx = W.ra_regex(n)
    alpha = DIGITS + b"a"
    sfa = P.SFA(rx, alpha)
    d = O.OracleDFA(rx, alpha)
    a = W.ra_text(16 << 20)
    assert sfa.match(torch.from_numpy(a).cuda()) == d.run(a)
    assert d.run(a)[1] is True
    mixed = np.concatenate([W.rn_accepted(n, 1 << 20), a[:1000]])
    assert sfa.match(torch.from_numpy(mixed).cuda()) == d.run(mixed)
    assert d.run(mixed)[1] is False
