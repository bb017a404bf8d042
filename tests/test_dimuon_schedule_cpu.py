"""Host-side model of the carried-list schedule of k_dimuon_carry (csrc/gvx_kernels.cuh,
dimuon_carry_tiles): per CTA iteration, phase A appends the tile's selected
entries at the list tail, phase B consumes the entries appended BEFORE this iteration's
selection in full passes of NT entries (everything on the final, tile-less iteration).

Checked for random selection counts (0..ET per tile, including the all-selected worst case):
every entry is consumed exactly once and in order, no pass is partial except the last one,
and the live span (tail - head) never exceeds the 2 ET + NT bound that sizes the circular
list (DimuonCarry<ET, NT>::CAP, the next power of two), so a slot is never overwritten
while still unconsumed. No GPU needed."""
import numpy as np
import pytest


def cap_of(et, nt):
    need = 2 * et + nt
    c = 1024
    while c < need:
        c *= 2
    return c


def run_schedule(counts, nt):
    """counts[i]: entries selected in the CTA's i-th tile. Returns (consumed order, max live
    span, pass sizes)."""
    head = mark = tail = 0
    consumed, passes, max_live = [], [], 0
    i = 0
    while True:
        have = i < len(counts)
        if have:
            tail += counts[i]  # phase A: appends at the tail
        max_live = max(max_live, tail - head)
        avail = (mark if have else tail) - head  # phase B: entries older than this selection
        take = (avail // nt) * nt if have else avail
        mark = tail
        for j0 in range(0, take, nt):
            passes.append(min(nt, take - j0))
        consumed.extend(range(head, head + take))
        head += take
        if not have:
            break
        i += 1
    return consumed, max_live, passes, tail


@pytest.mark.parametrize("et,nt", [(1024, 128), (2048, 256), (512, 128), (1024, 256)])
def test_carried_list_schedule(et, nt):
    rng = np.random.default_rng(et + nt)
    cap = cap_of(et, nt)
    for trial in range(200):
        ntiles = int(rng.integers(0, 40))
        mode = trial % 4
        if mode == 0:
            counts = rng.integers(0, et + 1, ntiles)          # anything
        elif mode == 1:
            counts = np.full(ntiles, et)                      # every event selected
        elif mode == 2:
            counts = rng.binomial(et, 0.15, ntiles)           # the recipe's ~15 %
        else:
            counts = rng.integers(0, 3, ntiles)               # almost nothing selected
        consumed, max_live, passes, total = run_schedule([int(c) for c in counts], nt)
        assert consumed == list(range(total))                 # each entry once, in order
        assert max_live <= 2 * et + nt - 1                    # (NT - 1) carried + two tiles
        assert max_live <= cap                                 # the circular list never wraps onto live slots
        assert all(p == nt for p in passes[:-1])               # only the final drain pass may be partial
        assert not passes or 0 < passes[-1] <= nt


def test_capacity_bound_is_tight():
    """The worst case (every event selected, NT - 1 entries carried) reaches 2 ET + NT - 1."""
    et, nt = 1024, 128
    counts = [nt - 1] + [et] * 5
    _, max_live, _, _ = run_schedule(counts, nt)
    assert max_live == 2 * et + nt - 1
    assert cap_of(et, nt) >= max_live
