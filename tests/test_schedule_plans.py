"""Host-side schedule plans of libeqc (eqc_comm.h), checked on the CPU.

Direct send: n balanced row bands (R-C13), one
band per rank; message pattern of fDirectSend: each of n ranks sends n-1
colour+depth tiles, the destination assembles n-1 colour tiles,
i.e. n(n-1) + (n-1) messages.  Binary swap: log2 n
rounds with partner rank ^ 2^r; final regions partition the frame in
bit-reversed order; non-power-of-two n is unsupported.
"""
import numpy as np
import pytest

from paper_1902_08755_b200 import eqc


@pytest.mark.parametrize("h,n", [(1080, 1), (1080, 2), (1081, 3), (2160, 4), (7, 8), (3, 5), (4320, 8)])
def test_bands_partition_and_balance(h, n):
    row0 = eqc.eqc_plan_bands(h, n)
    assert row0[0] == 0 and row0[-1] == h and len(row0) == n + 1
    sizes = [row0[j + 1] - row0[j] for j in range(n)]
    assert all(s >= 0 for s in sizes)
    assert max(sizes) - min(sizes) <= 1
    assert row0 == [j * h // n for j in range(n + 1)]


@pytest.mark.parametrize("h,n,dest", [(2160, 3, 0), (2160, 4, 0), (4320, 4, 3), (1081, 5, 2), (2160, 8, 0),
                                        (7, 8, 7), (1080, 2, 0), (1080, 1, 0)])
def test_gather_bands_balance_the_links(h, n, dest):
    """Gather-aware bands (R-C13 refinement, >= 3 ranks): a partition of the
    rows in rank order; the destination's band is round(h / (2n - 1)); the
    others differ by at most one row; every rank's NVLink inbound -- band
    pulls of 8 B/px from each peer plus, at the destination, the other bands'
    colour (4 B/px) -- is within one row's worth of the others'."""
    row0 = eqc.eqc_plan_bands_gather(h, n, dest)
    assert row0[0] == 0 and row0[-1] == h and len(row0) == n + 1
    sizes = [row0[j + 1] - row0[j] for j in range(n)]
    assert all(s >= 0 for s in sizes)
    if n <= 2:
        assert row0 == eqc.eqc_plan_bands(h, n)
        return
    assert sizes[dest] == (h + (2 * n - 1) // 2) // (2 * n - 1)
    others = [s for j, s in enumerate(sizes) if j != dest]
    assert max(others) - min(others) <= 1
    inbound = [8 * (n - 1) * s + (4 * (h - s) if j == dest else 0) for j, s in enumerate(sizes)]
    # unequal bands trade one rank's excess against the others: at most a
    # few rows' worth of imbalance remains from the rounding
    assert max(inbound) - min(inbound) <= 8 * (n - 1) * 2 + 4 * 2
    # and the destination receives less than with equal bands
    eq = eqc.eqc_plan_bands(h, n)
    eq_dest = eq[dest + 1] - eq[dest]
    assert inbound[dest] < 8 * (n - 1) * eq_dest + 4 * (h - eq_dest)


def bitrev(x, k):
    return int(format(x, f"0{k}b")[::-1], 2) if k else 0


@pytest.mark.parametrize("h,n", [(1080, 1), (1080, 2), (1081, 4), (4320, 8), (5, 8), (2160, 16)])
def test_binary_swap_plan(h, n):
    k = n.bit_length() - 1
    plans = [eqc.eqc_plan_binary_swap(h, n, r) for r in range(n)]
    assert all(len(p) == k for p in plans)  # log2 n rounds (n = 4 -> 2 rounds)
    for r in range(n):
        for rd, (partner, low, ky0, ky1, sy0, sy1) in enumerate(plans[r]):
            assert partner == r ^ (1 << rd)
            assert low == int(((r >> rd) & 1) == 0)
            p = plans[partner][rd]
            # the partner keeps exactly what I send and sends what I keep
            assert (p[2], p[3]) == (sy0, sy1) and (p[4], p[5]) == (ky0, ky1)
            # the kept half of the low rank is the upper rows
            if low:
                assert ky0 <= ky1 == sy0 <= sy1
            else:
                assert sy0 <= sy1 == ky0 <= ky1
    finals = []
    for r in range(n):
        y0, y1 = (plans[r][-1][2], plans[r][-1][3]) if k else (0, h)
        finals.append((y0, y1, r))
    finals.sort()
    # final regions tile [0, h) with no overlap, in bit-reversed rank order
    pos = 0
    for y0, y1, r in finals:
        assert y0 == pos
        pos = y1
    assert pos == h
    if h >= n:
        assert [r for _, _, r in finals] == [bitrev(i, k) for i in range(n)]


def test_binary_swap_rejects_non_power_of_two():
    with pytest.raises(eqc.EqcError) as e:
        eqc.eqc_plan_binary_swap(100, 3, 0)
    assert e.value.code == eqc.E_UNSUPPORTED


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_direct_send_message_count(n):
    """n(n-1) band exchanges + (n-1) gathers; for n = 3: two
    colour+depth tiles sent per channel, two colour tiles assembled at the
    destination."""
    row0 = eqc.eqc_plan_bands(2160, n)
    band_msgs = sum(1 for me in range(n) for j in range(n) if j != me and row0[j + 1] > row0[j])
    gathers = sum(1 for q in range(n) if q != 0 and row0[q + 1] > row0[q])
    assert band_msgs == n * (n - 1)
    assert gathers == n - 1


# ---- 2-3 swap plans (R-C21) ----------------------------------
def _s23_plans(h, n):
    return [eqc.eqc_plan_swap23(h, n, r) for r in range(n)]


@pytest.mark.parametrize("n", list(range(1, 21)) + [24, 27, 36])
def test_swap23_final_regions_partition_the_frame(n):
    for h in (1, 7, 100, 1081):
        plans = _s23_plans(h, n)
        covered = np.zeros(h, int)
        for p in plans:
            y0, y1 = p["final"]
            if p["fold_role"] == 2:
                assert (y0, y1) == (0, 0) and not p["rounds"]
            covered[y0:y1] += 1
        assert (covered == 1).all()  # every row owned by exactly one rank


@pytest.mark.parametrize("n", list(range(1, 21)) + [24, 27, 36])
def test_swap23_groups_of_two_or_three_consistent(n):
    h = 720
    plans = _s23_plans(h, n)
    for p in plans:
        for r, rd in enumerate(p["rounds"]):
            assert rd["k"] in (2, 3) and len(rd["members"]) == rd["k"]
            assert rd["members"] == sorted(rd["members"])
            for u, q in enumerate(rd["members"]):  # every member agrees on the group
                other = plans[q]["rounds"][r]
                assert other["members"] == rd["members"] and other["bounds"] == rd["bounds"]
                assert other["t"] == u
    folds = [p for p in plans if p["fold_role"]]
    for r, p in enumerate(plans):
        if p["fold_role"]:
            assert plans[p["fold_partner"]]["fold_partner"] == r
            assert {p["fold_role"], plans[p["fold_partner"]]["fold_role"]} == {1, 2}
    assert len(folds) % 2 == 0


@pytest.mark.parametrize("n", list(range(1, 21)) + [24, 27, 36])
def test_swap23_symbolic_execution_reaches_all_sources_in_order(n):
    # track, per rank and row, the ordered list of source ranks composited so
    # far: every final row must hold ALL ranks, merged in ascending order
    h = 97
    plans = _s23_plans(h, n)
    held = {r: [[r] for _ in range(h)] for r in range(n)}
    for r, p in enumerate(plans):
        if p["fold_role"] == 1:
            q = p["fold_partner"]
            held[r] = [a + b for a, b in zip(held[r], held[q])]
    nr = max(len(p["rounds"]) for p in plans)
    for rd in range(nr):
        new = {r: [list(x) for x in held[r]] for r in range(n)}
        for r, p in enumerate(plans):
            if rd >= len(p["rounds"]):
                continue
            R = p["rounds"][rd]
            y0, y1 = R["bounds"][R["t"]], R["bounds"][R["t"] + 1]
            for y in range(y0, y1):
                new[r][y] = sum((held[q][y] for q in R["members"]), [])
        held = new
    for r, p in enumerate(plans):
        y0, y1 = p["final"]
        for y in range(y0, y1):
            assert held[r][y] == list(range(n)), (n, r, y)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
def test_swap23_is_binary_swap_for_powers_of_two(n):
    h = 1081
    for r in range(n):
        p = eqc.eqc_plan_swap23(h, n, r)
        bs = eqc.eqc_plan_binary_swap(h, n, r)
        assert p["fold_role"] == 0 and len(p["rounds"]) == len(bs)
        for rd, b in zip(p["rounds"], bs):
            partner, low, ky0, ky1, sy0, sy1 = b
            assert rd["k"] == 2 and partner in rd["members"]
            assert (rd["bounds"][rd["t"]], rd["bounds"][rd["t"] + 1]) == (ky0, ky1)
            assert (rd["t"] == 0) == bool(low)
