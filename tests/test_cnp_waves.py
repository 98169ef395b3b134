"""Host logic of the CNP wave launches (trainer.cnp_wave_*): the forward's
launches extend a computed prefix that always covers the decoder block
about to run, in whole waves; the backward's launches partition the stack
from the top, each (but the last) a whole number of waves, and never
include a block whose dG is not ready."""

import itertools

import pytest

from paper_2603_05500_b200.trainer import cnp_wave_bwd_start, cnp_wave_fwd_target


def ranges(sizes):
    out, off = [], 0
    for n in sizes:
        out.append((off, n))
        off += n
    return out


@pytest.mark.parametrize("sizes,wave", [([154] * 24, 74), ([77] * 24, 74), ([154] * 32, 74), ([40] * 3, 74),
                                        ([154] * 24, 148), ([5, 300, 7, 74, 1], 74), ([154] * 24, 1)])
def test_cnp_wave_launches(sizes, wave):
    br = ranges(sizes)
    nb = sum(sizes)
    # forward: before decoder block i runs, blocks < its end are computed
    done, launches = 0, []
    for off, n in br:
        tgt = cnp_wave_fwd_target(off + n, done, wave, nb)
        if tgt > done:
            launches.append((done, tgt))
        done = tgt
        assert done >= off + n
    assert done == nb
    assert all((b - a) % wave == 0 for a, b in launches[:-1])
    # backward: hooks fire top block first; launch [start, hi) with blocks >= off ready
    hi, covered = nb, []
    for i in reversed(range(len(br))):
        off = br[i][0]
        start = cnp_wave_bwd_start(off, hi, wave, i == 0)
        assert start >= off  # only ready blocks
        if start < hi:
            covered.append((start, hi))
            if i != 0:
                assert (hi - start) % wave == 0
            hi = start
    assert hi == 0
    flat = sorted(itertools.chain.from_iterable(range(a, b) for a, b in covered))
    assert flat == list(range(nb))
