"""The TMA scan plan (csrc/plan.hpp make_plan), host logic, no GPU: compiled
with g++ against the same header the kernels and the device-side batch planner
use, and checked on many sizes and alignments.

Invariants: the head brings the rows to 256-B alignment; the rows are cut at
multiples of L (a multiple of 64, >= 256) and the pieces head | rows | tail
tile [0, n) exactly (every byte is read once); every CTA
gets ceil or floor of rows / G rows (all G SMs scan once there are G rows),
loaded as at most NB TMA boxes per stage (full boxes of bh rows, bh a multiple
of 8 and <= 256, then one partial box); the tail is less than one row."""
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
    // stdin: addr n G R NB rowb align [len: equal texts of len bytes, n = their count] ; stdout: the plan fields
    unsigned long long addr, n, len; unsigned G, R, NB, rowb, al;
    while (scanf("%llu %llu %u %u %u %u %u %llu", &addr, &n, &G, &R, &NB, &rowb, &al, &len) == 8) {
        sfa::TmaPlan p;
        if (len) {
            if (!sfa::make_plan_uniform(addr, len, n, G, R, NB, rowb, &p)) { printf("none\n"); continue; }
        } else {
            sfa::make_plan(addr, n, G, R, NB, rowb, al, &p);
        }
        printf("%llu %llu %u %u %u %u %u %u %llu\n", (unsigned long long)p.head, (unsigned long long)p.L,
               p.nchunks, p.ctas, p.rc_hi, p.rc_lo, p.m, p.bh, (unsigned long long)p.tail_start);
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
        inp = "".join(" ".join(str(x) for x in (c if len(c) == 8 else (*c, 0))) + "\n" for c in cases)
        out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
        return [None if line.strip() == "none" else tuple(int(x) for x in line.split()) for line in out if line.strip()]
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
    for (addr, n, G, R, NB, rowb, al), (head, L, rows, ctas, hi, lo, m, bh, tail) in zip(cases, out):
        assert head < 256 and head <= n
        if head < n:
            assert (addr + head) % 256 == 0
        assert L >= 256 and L % 64 == 0 and L % rowb == 0
        if al:
            assert L % al == 0
        assert tail == head + rows * L and tail <= n and n - tail < max(L, 256)   # the tail is < one row
        assert rows <= G * R
        if rows == 0:
            continue
        assert 1 <= ctas <= G and hi <= R and hi - lo <= 1
        assert bh % 8 == 0 and 8 <= bh <= 256 and hi <= NB * bh       # <= NB boxes per stage
        per = [hi if b < m else lo for b in range(ctas)]
        assert sum(per) == rows and min(per) >= 1                     # the split tiles the rows exactly
        assert max(per) == -(-rows // G)                              # busiest CTA: the ceiling of the average
        if rows >= G:
            assert ctas == G


def test_plan_uses_every_sm_on_the_configs(planner):
    """cfg2 (256 MiB) and the 1 GiB / 4 GiB ranges: all 148 SMs get rows and
    the busiest carries < 1% more than the average (round 1 left 2 idle)."""
    for n in (268_435_450, 1 << 30, 1 << 32):
        (head, L, rows, ctas, hi, lo, m, bh, tail), = planner([(0x7f0000000000, n, 148, 992, 4, 32, 0)])
        assert ctas == 148
        assert hi * L <= n / 148 + L


def test_plan_equal_texts(planner):
    """Equal texts (make_plan_uniform): every text is mm whole rows (no text
    boundary inside a row), the rows tile the batch exactly, no head or tail;
    refused for unaligned bases, lengths that no row length divides, and
    batches whose texts outnumber the rows."""
    cases = [(0x7f0000000000, 65536, 148, 992, 4, 16, 0, 65536), (0x7f0000000000, 300, 148, 992, 4, 32, 0, 65536),
             (0x7f0000000000, 5000, 148, 1984, 8, 32, 0, 4096), (0x7f0000000020, 777, 148, 992, 4, 32, 0, 1024),
             (0x7f0000000010, 300, 148, 992, 4, 32, 0, 65536), (0x7f0000000000, 100, 148, 992, 4, 32, 0, 1000),
             (0x7f0000000000, 200_000, 148, 992, 4, 32, 0, 256), (0x7f0000000000, 3, 148, 992, 4, 16, 0, 1 << 24), (0x7f0000000000, 146816, 148, 992, 4, 16, 0, 256)]
    out = planner(cases)
    for (addr, count, G, R, NB, rowb, _, ln), o in zip(cases, out):
        if addr % 32 or ln % 16 or count > G * R or ln < 256:
            assert o is None, (addr, count, ln)
            continue
        head, L, rows, ctas, hi, lo, m, bh, tail = o
        assert head == 0 and ln % L == 0 and L % rowb == 0 and L >= 256 and rows == count * (ln // L)
        assert tail == count * ln
        assert rows <= G * R and hi - lo <= 1 and hi <= NB * bh
    assert out[0][1] == 32768          # cfg5: two rows of 32 KiB per 64 KiB text


MIX_SRC = r'''
#include <cstdio>
#include <set>
#include "plan.hpp"
// The MIXED DFA-window encoding (plan.hpp mix_*), the 16-byte fix and the
// compact source expansion: prints "ok" or the first violated property.
int main() {
    const unsigned Hs[] = {2, 8, 68, 70, 100}, nDs[] = {101, 145, 300, 513};
    for (unsigned H : Hs)
        for (unsigned nD : nDs) {
            if (H >= nD) continue;
            const unsigned hotb = 64 * H, X = sfa::mix_X(nD, H);
            if (X % 128) { printf("X %u not a multiple of 128\n", X); return 0; }
            std::set<unsigned> seen;
            for (unsigned r = 0; r < H; ++r)
                for (unsigned L = 0; L < 32; ++L) {
                    const unsigned e = sfa::mix_hot(r, L);
                    if (e + 2 > hotb) { printf("hot %u,%u outside the hot region\n", r, L); return 0; }
                    if ((e >> 2) % 32 != L) { printf("hot %u,%u not in bank %u\n", r, L, L); return 0; }
                    if (!seen.insert(e).second) { printf("hot %u,%u shares a cell\n", r, L); return 0; }
                    if (sfa::mix_rank_of(e, hotb) != r) { printf("rank of hot %u,%u\n", r, L); return 0; }
                    if (sfa::mix_fix(e, hotb, 4 * L) != e) { printf("fix moved hot %u,%u\n", r, L); return 0; }
                    for (unsigned j = 1; j < 4; ++j)  // other columns keep the bank
                        if (((j * X + e) >> 2) % 32 != L) { printf("column %u moves bank\n", j); return 0; }
                }
            for (unsigned r = 0; r < nD; ++r) {
                const unsigned t = sfa::mix_twin(r, hotb, H);
                if (r < H) {  // a hot state's twin is lane 31's private cell
                    if (t != sfa::mix_hot(r, 31)) { printf("twin of hot %u is not lane 31's cell\n", r); return 0; }
                } else {
                    if (t < hotb || t + 2 > X) { printf("twin %u outside the twin region\n", r); return 0; }
                    if (!seen.insert(t).second) { printf("twin %u shares a cell\n", r); return 0; }
                }
                if (sfa::mix_rank_of(t, hotb) != r) { printf("rank of twin %u\n", r); return 0; }
                for (unsigned L = 0; L < 32; L += 7) {
                    const unsigned f = sfa::mix_fix(t, hotb, 4 * L);
                    if (f != (r < H ? sfa::mix_hot(r, L) : t)) { printf("fix of twin %u lane %u\n", r, L); return 0; }
                }
            }
            if (X > 32768) continue;  // the compact source needs values < 2^15
            for (unsigned a = 0; a < nD; a += 3)
                for (unsigned b = 0; b < nD; b += 5) {
                    auto cell = [&](unsigned q) {
                        return q < H ? sfa::cpt_cell(sfa::mix_hot(q, 0), true) : sfa::cpt_cell(sfa::mix_twin(q, hotb, H), false);
                    };
                    auto enc = [&](unsigned q, unsigned L) { return q < H ? sfa::mix_hot(q, L) : sfa::mix_twin(q, hotb, H); };
                    for (unsigned L = 0; L < 32; ++L)
                        if (sfa::cpt_expand(cell(a) | (cell(b) << 16), L) != (enc(a, L) | (enc(b, L) << 16))) {
                            printf("compact expansion %u %u lane %u\n", a, b, L);
                            return 0;
                        }
                }
        }
    printf("ok\n");
}
'''


def test_mixed_window_encoding(tmp_path):
    """MIXED DFA window (plan.hpp): lane L's private cells of the hot states
    all sit in bank L in every column, no two cells of the layout coincide,
    ranks decode from both encodings, a hot state's twin is lane 31's private
    cell, the 16-byte fix sends exactly the twins of hot states to the lane's
    own cell, and the compact source
    (bit 15 = private target) expands to every lane's pair word."""
    src = tmp_path / "mix.cpp"
    src.write_text(MIX_SRC)
    exe = tmp_path / "mix"
    csrc = os.path.join(ROOT, "paper_1405_0562_b200", "csrc")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I", csrc, "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", str(src), "-o", str(exe)])
    assert subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.strip() == "ok"
