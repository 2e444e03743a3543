"""Scripted pins of the oracle's lane-change, gap-acceptance, stop-within-step
and conflict arithmetic (-m "not gpu").

Each case puts vehicles at a chosen snapshot (``Oracle.set_state``) and checks
the next snapshot against values fixed outside the oracle:

* the SURVEY.md §8(c) worked cases (SURVEY.md:583 merge timeline, :584 lane
  change, :585 ε values), computed in an independent session;
* gap acceptance with a non-free target lane — Eq. (Gap Acceptance)
  PAPER.md:228-235 (§3.2), reading Q15/Q17 — with the expected
  accept / reject decided from g_lead / g_lag evaluated here in fp64 from the
  KAT-pinned test-side Philox words, and cases built with margins so that a
  sign error in an anticipation term (α_a, α_b, α_i) flips the decision;
* the stop-within-step branch of the kinematics — Alg. 1, reading
  Q11: dx = v²/(2|acc|) — against the IDM closed form in fp64.

Mutation check (run by hand when this file was written, see the commit): a
flipped sign of the α_a term in the oracle's g_lead, a flipped α_b term in
g_lag, or a dropped ½ in the stop branch each turn at least one test here red.
"""
import math

import numpy as np
import pytest

from tests.helpers import demand_from_routes, graph_from_edges, lc_network, merge_network, philox4x32_10

SIGMA = 0.5
DT = 0.5
A, B, S0, T = 1.5, 2.0, 2.0, 1.5


def place(oracle_mod, g, routes, state, step=0, params=None, depart=None):
    """routes: per trip; state: {id: (edge, lane, pos, v, cursor)}; other trips wait (depart late)."""
    n = len(routes)
    dep = depart if depart is not None else [1.0e5] * n
    o = oracle_mod.Oracle(g, params)
    o.load_demand(**demand_from_routes(routes, dep))
    status = np.zeros(n, np.int32)
    edge = np.array([r[0] for r in routes], np.int32)
    lane = np.zeros(n, np.int32)
    pos = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    cur = np.zeros(n, np.int64)
    for i, (e, l, p, sp, j) in state.items():
        status[i], edge[i], lane[i], pos[i], v[i], cur[i] = 1, e, l, p, sp, j
    o.set_state(step, status, edge, lane, pos, v, cur)
    return o


def test_set_state_roundtrip(oracle_mod):
    g = lc_network(length=200.0)
    routes = [[3, 0]] * 7 + [[0, 1], [0, 1]]
    o = place(oracle_mod, g, routes, {7: (0, 1, 20.5, 10.0, 0), 8: (0, 0, 40.25, 3.0, 0)}, step=11)
    st = o.trip_state()
    assert st["status"].tolist() == [0] * 7 + [1, 1]
    assert st["pos"][7] == np.float32(20.5) and st["lane"][8] == 0
    m = o.lane_map()
    assert int((m != 255).sum()) == 2 and m[200 + 20] == 10 and m[40] == 3  # lane 1 starts at Lc = 200
    assert o.stats()["step"] == 11
    with pytest.raises(oracle_mod.OracleError):  # two vehicles in one byte
        place(oracle_mod, g, routes, {7: (0, 0, 20.5, 1.0, 0), 8: (0, 0, 20.9, 1.0, 0)})


# ---------------------------------------------------------------------------
# SURVEY.md:585 — ε values (σ = 0.5, seed 1), computed in the survey session
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("tid,k,stream,want", [(0, 0, 1, -0.9194477), (0, 0, 2, -0.2259700), (7, 0, 1, -0.6162567)])
def test_eps_survey_values(oracle_mod, tid, k, stream, want):
    assert abs(oracle_mod.eps(1, tid, k, stream, SIGMA) - want) < 5e-7


# ---------------------------------------------------------------------------
# SURVEY.md:583 — merge timeline (Remark "Switch"; lowest id wins, A9)
# ---------------------------------------------------------------------------
def test_merge_worked_timeline(oracle_mod):
    g = merge_network(len_in=100.0)
    routes = [[3, 0]] * 6
    routes[3], routes[5] = [0, 2], [1, 2]
    o = place(oracle_mod, g, routes, {3: (0, 0, 99.95, 0.0, 0), 5: (1, 0, 99.95, 0.0, 0)})
    hist = []
    for _ in range(30):
        o.step(1)
        st = o.trip_state()
        hist.append({i: (int(st["edge"][i]), int(st["cursor"][i]), float(st["pos"][i]), float(st["v"][i]))
                     for i in (3, 5)})
    # snapshot 1: id 3 won cell 0 of the out-edge (pos 0, v 0.75); id 5 fell back to 99.95, v 0
    assert hist[0][3] == (2, 1, 0.0, 0.75)
    assert hist[0][5] == (1, 0, np.float32(99.95), 0.0)
    # snapshots 1-4: id 5 holds at the line (s = 1, 1, 2 = s0 -> acc <= 0; then the road looks free)
    for m in range(4):
        assert hist[m][5][:2] == (1, 0) and hist[m][5][3] == 0.0
    assert abs(hist[2][3][2] - 1.49997) < 2e-5  # id 3 in cell 1 at snapshot 3
    # snapshot 5: id 5 enters (pos 0, v 0.75) and then follows id 3 exactly 4 steps behind
    assert hist[4][5] == (2, 1, 0.0, 0.75)
    for m in range(0, 20):
        assert hist[4 + m][5][2:] == hist[m][3][2:]


# ---------------------------------------------------------------------------
# SURVEY.md:584 — lane-change worked case (Eq. Lane Change PAPER.md:222-225)
# ---------------------------------------------------------------------------
def test_lane_change_worked_values(oracle_mod):
    g = lc_network(length=100.0)
    routes = [[3, 0]] * 7 + [[0, 1]]
    o = place(oracle_mod, g, routes, {7: (0, 1, 20.0, 10.0, 0)})
    u = [(philox4x32_10((7, k, 0, 0), (1, 0))[0] >> 8) / 2.0**24 for k in range(3)]
    assert abs(u[0] - 0.480692) < 1e-6 and abs(u[1] - 0.875646) < 1e-6 and abs(u[2] - 0.139313) < 1e-6
    lanes, pos = [], []
    for _ in range(3):
        o.step(1)
        st = o.trip_state()
        lanes.append(int(st["lane"][7]))
        pos.append(float(st["pos"][7]))
    # free road at v = 10: acc 1.09818, dx 5.13727 (fp64 closed form)
    acc = A * (1 - (10 / 13.9) ** 4)
    assert abs(pos[0] - (20 + 10 * DT + 0.5 * acc * DT**2)) < 2e-5
    assert abs((100 - (100 - pos[0])) / 100 - 0.251373) < 2e-6
    assert lanes == [1, 1, 0]
    assert abs(pos[2] - 36.17487) < 5e-5
    assert o.stats()["lane_changes"] == 1


# ---------------------------------------------------------------------------
# Gap acceptance with a lead and a lag in the target lane (Eq. Gap Acceptance,
# PAPER.md:228-235; Q15 form, Q17 lag bound) — expected decisions in fp64
# ---------------------------------------------------------------------------
def eps64(tid, k, stream, sigma=SIGMA):
    """Q15: ε = σ√3 (Σ_j (x_j >> 10) 2^-22 − 2) from the KAT-pinned test-side Philox, in fp64."""
    w = philox4x32_10((tid, k, stream, 0), (1, 0))
    return sigma * math.sqrt(3.0) * (sum(x >> 10 for x in w) * 2.0**-22 - 2.0)


def u64(tid, k):
    return (philox4x32_10((tid, k, 0, 0), (1, 0))[0] >> 8) / 2.0**24


def free_pos(p, v, v0=13.9):
    acc = A * (1 - (v / v0) ** 4)
    return p + v * DT + 0.5 * acc * DT**2


def expect_accept(v, lead, lag, k, tid=7):
    """lead/lag: (gap in cells, byte) or None.  g_lead = max(0, g_a + α_i v − α_a b_ld + ε_a),
    g_lag = max(0, g_b + α_b b_lg − α_i v + ε_b), lag kinematic bound S(b) = ceil((b+1)Δt + ½aΔt²) + 1."""
    ok = True
    if lead is not None:
        g_lead = max(0.0, 2.0 + 0.5 * v - 0.5 * lead[1] + eps64(tid, k, 1))
        ok = ok and lead[0] >= g_lead
    if lag is not None:
        g_lag = max(0.0, 2.0 + 0.5 * lag[1] - 0.5 * v + eps64(tid, k, 2))
        S = math.ceil((lag[1] + 1) * DT + 0.5 * A * DT**2) + 1
        ok = ok and lag[0] >= g_lag and lag[0] >= S
    return ok


def lc_scene(oracle_mod, v, lead, lag, p=150.3, k=None):
    """Trip 7 in lane 1 of a 200 m 2-lane edge must move to lane 0 (toward e1, allowed [0,0]);
    trip 8 = lead, trip 9 = lag in lane 0 at the given gaps from 7's new cell c'.  The step k is the
    first with u(7, k) < p_LC so the change is attempted.  Returns (lane of 7 at k+1, c', k)."""
    g = lc_network(length=200.0)
    plc = (100.0 - (200.0 - p)) / 100.0
    if k is None:
        k = next(kk for kk in range(1000) if u64(7, kk) < plc)
    pn = free_pos(p, v)
    assert abs(pn - round(pn)) > 1e-3, "scene too close to a cell boundary"
    cn = math.floor(pn)
    state = {7: (0, 1, p, v, 0)}
    if lead is not None:
        state[8] = (0, 0, cn + lead[0] + 0.5, lead[1] + 0.5, 0)
    if lag is not None:
        state[9] = (0, 0, cn - lag[0] + 0.25, lag[1] + 0.25, 0)
    routes = [[3, 0]] * 7 + [[0, 1], [0, 1], [0, 1]]
    o = place(oracle_mod, g, routes, state, step=k)
    o.step(1)
    st = o.trip_state()
    assert st["edge"][7] == 0 and math.floor(st["pos"][7]) == cn
    return int(st["lane"][7]), cn, k


def test_lead_anticipation_sign(oracle_mod):
    """v = 10, lead byte 12 three cells ahead: g_lead = 2 + 5 − 6 + ε_a = 1 + ε_a < 3 for every ε_a
    (|ε| < 2√3σ = 1.73): accepted.  A wrong sign of the α_a term (+6) would give 13 + ε_a: rejected."""
    lane, _, k = lc_scene(oracle_mod, 10.0, (3, 12), None)
    assert expect_accept(10.0, (3, 12), None, k)
    assert lane == 0


def test_lead_rejects_slow_leader(oracle_mod):
    """v = 10, lead byte 2 four cells ahead: g_lead = 6 + ε_a > 4.27 > 4: rejected for every ε_a."""
    lane, _, k = lc_scene(oracle_mod, 10.0, (4, 2), None)
    assert not expect_accept(10.0, (4, 2), None, k)
    assert lane == 1


@pytest.mark.parametrize("v,b_ld", [(10.0, 6), (6.0, 3), (12.0, 9)])
def test_lead_gap_threshold(oracle_mod, v, b_ld):
    """At the fp64 threshold: gap = ceil(g_lead) is accepted, ceil(g_lead) − 1 rejected."""
    p = 150.3
    plc = (100.0 - (200.0 - p)) / 100.0
    k = next(kk for kk in range(1000) if u64(7, kk) < plc)
    g_lead = max(0.0, 2.0 + 0.5 * v - 0.5 * b_ld + eps64(7, k, 1))
    assert abs(g_lead - round(g_lead)) > 1e-3
    hi = max(1, math.ceil(g_lead))
    assert lc_scene(oracle_mod, v, (hi, b_ld), None, p=p, k=k)[0] == 0
    if hi - 1 >= 1:
        assert lc_scene(oracle_mod, v, (hi - 1, b_ld), None, p=p, k=k)[0] == 1


def test_lag_kinematic_bound(oracle_mod):
    """Lag byte 10: S(10) = ceil(11·0.5 + 0.1875) + 1 = 7 (SURVEY.md:584).  v = 10 gives
    g_lag = 2 + 5 − 5 + ε_b < 3.8: six cells are rejected by S alone, seven accepted."""
    assert math.ceil(11 * 0.5 + 0.1875) + 1 == 7
    lane6, _, k = lc_scene(oracle_mod, 10.0, None, (6, 10))
    assert not expect_accept(10.0, None, (6, 10), k) and lane6 == 1
    lane7, _, k = lc_scene(oracle_mod, 10.0, None, (7, 10))
    assert expect_accept(10.0, None, (7, 10), k) and lane7 == 0


def test_lag_anticipation_terms(oracle_mod):
    """v = 1, lag byte 20 at S(20) = 12 cells: g_lag = 2 + 10 − 0.5 + ε_b = 11.5 + ε_b.  Steps k are
    chosen where ε_b > 0.6 (rejected: g_lag > 12) and where ε_b < 0.4 (accepted).  A wrong sign of
    α_b (−10) or of α_i (+0.5 instead of −0.5 changes g_lag by 1) flips one of the two."""
    v, p = 1.0, 150.3
    plc = (100.0 - (200.0 - p)) / 100.0
    ks = [kk for kk in range(4000) if u64(7, kk) < plc]
    k_rej = next(kk for kk in ks if eps64(7, kk, 2) > 0.6)
    k_acc = next(kk for kk in ks if eps64(7, kk, 2) < 0.4)
    S = math.ceil(21 * 0.5 + 0.1875) + 1
    assert S == 12
    assert not expect_accept(v, None, (12, 20), k_rej)
    assert expect_accept(v, None, (12, 20), k_acc)
    assert lc_scene(oracle_mod, v, None, (12, 20), p=p, k=k_rej)[0] == 1
    assert lc_scene(oracle_mod, v, None, (12, 20), p=p, k=k_acc)[0] == 0


def test_lead_and_lag_together(oracle_mod):
    """Both sides present: accepted only if both critical gaps hold (fp64 expectation over several k)."""
    v, p = 8.0, 150.3
    plc = (100.0 - (200.0 - p)) / 100.0
    ks = [kk for kk in range(400) if u64(7, kk) < plc][:6]
    seen = set()
    for k in ks:
        for lead, lag in [((3, 8), (7, 9)), ((5, 4), (8, 10)), ((2, 3), (9, 6))]:
            want = expect_accept(v, lead, lag, k)
            g_lead = 2.0 + 0.5 * v - 0.5 * lead[1] + eps64(7, k, 1)
            g_lag = 2.0 + 0.5 * lag[1] - 0.5 * v + eps64(7, k, 2)
            if min(abs(g_lead - lead[0]), abs(g_lag - lag[0])) < 1e-3:
                continue
            lane = lc_scene(oracle_mod, v, lead, lag, p=p, k=k)[0]
            assert lane == (0 if want else 1), (k, lead, lag)
            seen.add(want)
    assert seen == {True, False}


def test_no_change_into_occupied_target_cell(oracle_mod):
    """The target cell itself occupied in M_k: never a change (Q17; the lead scan starts past it)."""
    p, v = 150.3, 10.0
    plc = (100.0 - (200.0 - p)) / 100.0
    k = next(kk for kk in range(1000) if u64(7, kk) < plc)
    cn = math.floor(free_pos(p, v))
    g = lc_network(length=200.0)
    routes = [[3, 0]] * 7 + [[0, 1], [0, 1]]
    o = place(oracle_mod, g, routes, {7: (0, 1, p, v, 0), 8: (0, 0, cn + 0.5, 20.0, 0)}, step=k)
    o.step(1)
    assert o.trip_state()["lane"][7] == 1


# ---------------------------------------------------------------------------
# Stop within the step (Alg. 1 PAPER.md:314 kinematics, reading Q11)
# ---------------------------------------------------------------------------
def idm64(v, v0, s, vf):
    """Textbook IDM (Q3/Q4) in fp64: a[1 − (v/v0)^4 − (s*/s)²], s* = s0 + max(0, vT + vΔv/(2√(ab)))."""
    ss = S0 + max(0.0, v * T + v * (v - vf) / (2 * math.sqrt(A * B)))
    return A * (1 - (v / v0) ** 4 - (ss / s) ** 2)


@pytest.mark.parametrize("p,v,gap", [(50.3, 13.0, 3), (20.6, 5.0, 1), (70.1, 9.0, 4)])
def test_stop_within_step_closed_form(oracle_mod, p, v, gap):
    """A vehicle closing on a stopped leader brakes so hard that v + aΔt < 0: it stops within the
    step after dx = v²/(2|acc|) (the ballistic distance to standstill) and v' = 0."""
    g = graph_from_edges(2, [(0, 1, 100.0, 1, 13.9), (1, 0, 100.0, 1, 13.9)])
    c = math.floor(p)
    acc = idm64(v, 13.9, gap, 0)
    assert v + acc * DT < 0
    o = place(oracle_mod, g, [[0], [0]], {0: (0, 0, p, v, 0), 1: (0, 0, c + gap + 0.5, 0.0, 0)})
    o.step(1)
    st = o.trip_state()
    want = p + v * v / (2 * abs(acc))
    assert st["v"][0] == 0.0
    assert abs(float(st["pos"][0]) - want) < 2e-5, (float(st["pos"][0]), want)
    assert math.floor(want) < c + gap  # the no-overtake clamp is not what stopped it
