"""The TMA scan plan (csrc/plan.hpp make_plan), host logic, no GPU: compiled
with g++ against the same header the kernels and the device-side batch planner
use, and checked on many sizes and alignments.

Invariants: the head brings the rows to 256-B alignment; the rows are cut at
multiples of L (a multiple of 64, >= 256) and the pieces head | rows | tail
tile [0, n) exactly (every byte is read once); every CTA
gets rc_hi or rc_lo rows whose TMA boxes (NB per stage, heights multiples of
8 rows and <= 256) cover them exactly; all G SMs get rows once the text is big
enough (the uneven split), their loads differ by less than 8*NB rows; the
tail stays small."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

SRC = r'''
#include <cstdio>
#include <cstdlib>
#include "plan.hpp"
int main(int argc, char** argv) {
    // stdin: addr n G R NB rowb align ; stdout: the plan fields
    unsigned long long addr, n; unsigned G, R, NB, rowb, al;
    while (scanf("%llu %llu %u %u %u %u %u", &addr, &n, &G, &R, &NB, &rowb, &al) == 7) {
        sfa::TmaPlan p;
        sfa::make_plan(addr, n, G, R, NB, rowb, al, &p);
        printf("%llu %llu %u %u %u %u %u %u %u %u %llu\n", (unsigned long long)p.head, (unsigned long long)p.L,
               p.nchunks, p.ctas, p.rc_hi, p.rc_lo, p.m, p.bh, p.bl_hi, p.bl_lo, (unsigned long long)p.tail_start);
    }
}
'''


@pytest.fixture(scope="module")
def planner(tmp_path_factory):
    d = tmp_path_factory.mktemp("plan")
    src = d / "plan.cpp"
    src.write_text(SRC)
    exe = d / "plan"
    csrc = os.path.join(ROOT, "paper_1405_0562_b200", "csrc")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I", csrc, "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", str(src), "-o", str(exe)])

    def run(cases):
        inp = "".join(" ".join(str(x) for x in c) + "\n" for c in cases)
        out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
        return [tuple(int(x) for x in line.split()) for line in out if line.strip()]
    return run


SHAPES = [(992, 4, 32), (1984, 8, 32), (992, 4, 64), (1984, 8, 16), (992, 4, 16)]


def test_plan_invariants(planner):
    rng = np.random.default_rng(0)
    cases = []
    for n in [4 << 20, (4 << 20) + 1, 5_000_001, 10 * 148 * 992 + 7, 268_435_450, 1 << 30, (1 << 32) + 5, 12_345_678,
              65536, 70_001, 300, 0, 17]:
        for R, NB, rowb in SHAPES:
            for addr in (0x7f0000000000, 0x7f0000000005, 0x7f00000000f1):
                for al in (0, 64, 128, 256):
                    cases.append((addr, n, 148, R, NB, rowb, al))
    for _ in range(300):
        R, NB, rowb = SHAPES[int(rng.integers(0, len(SHAPES)))]
        cases.append((0x7f0000000000 + int(rng.integers(0, 4096)), int(rng.integers(0, 1 << 33)),
                      int(rng.integers(1, 160)), R, NB, rowb, 0))
    out = planner(cases)
    assert len(out) == len(cases)
    for (addr, n, G, R, NB, rowb, al), (head, L, rows, ctas, hi, lo, m, bh, bl_hi, bl_lo, tail) in zip(cases, out):
        assert head < 256 and head <= n
        if head < n:
            assert (addr + head) % 256 == 0
        assert L >= 256 and L % 64 == 0 and L % rowb == 0
        if al:
            assert L % al == 0
        assert tail == head + rows * L and tail <= n
        assert rows <= G * R
        if rows == 0:
            assert n - head < 256
            continue
        assert 1 <= ctas <= G
        assert hi <= R and hi % 8 == 0 and bh % 8 == 0 and 8 <= bh <= 256
        assert bl_hi % 8 == 0 and bl_lo % 8 == 0 and 8 <= bl_lo <= bl_hi <= 256
        assert (NB - 1) * bh + bl_hi == hi and (NB - 1) * bh + bl_lo == lo   # the boxes tile each CTA's rows
        # rows per CTA: m CTAs with hi rows, then lo rows
        per = [hi if b < m else lo for b in range(ctas)]
        if lo < hi:
            assert ctas == G and sum(per) == rows         # every SM scans; the split tiles the rows exactly
            assert hi - lo == 8
            assert hi * G - rows < 8 * G + 8 * G          # busiest CTA within 8 rows of the average
        else:
            assert m == ctas and (ctas - 1) * hi < rows <= ctas * hi   # last CTA's extra rows are TMA zero fill
        # the tail (plus the < 8 rows the split leaves over) stays below 8 rows
        assert n - tail < 8 * L + (L if lo == hi else 0)
        if n >= 64 * G * R:
            assert ctas == G and lo < hi


def test_plan_uses_every_sm_on_the_configs(planner):
    """cfg2 (256 MiB) and the 1 GiB / 4 GiB ranges: all 148 SMs get rows and
    the busiest carries < 1% more than the average (round 1 left 2 idle)."""
    for n in (268_435_450, 1 << 30, 1 << 32):
        (head, L, rows, ctas, hi, lo, m, bh, bl_hi, bl_lo, tail), = planner([(0x7f0000000000, n, 148, 992, 4, 32, 0)])
        assert ctas == 148
        assert hi * L <= 1.01 * n / 148 + L
