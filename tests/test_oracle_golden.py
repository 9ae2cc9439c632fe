"""Pin the CPU oracle (oracle/ref_oracle.py) to the reference's golden fixtures.

The fixtures come from calling the reference package itself
(tests/golden/make_golden.py); these tests prove the numpy restatement
reproduces its transforms, stage-strike layouts and every protected-run
decision before the oracle is trusted as the checker for the CUDA path.
"""

import hashlib

import numpy as np
import pytest

from conftest import gaussian, golden, golden_abft_outputs, golden_fft_outputs, max_rel_error, oracle_tol
from oracle import ref_oracle as O


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def faults_of(specs):
    return [O.Fault(**s) for s in specs]


@pytest.mark.parametrize("case", golden()["fft_cases"], ids=lambda c: c["name"])
def test_oracle_transform_matches_reference(case):
    x = gaussian(case["n"], case["b"], case["precision"], case["seed"])
    assert digest(x) == case["x_digest"], "input generator drifted"
    plan = O.Plan(tuple(case["spans"]), tuple(case["radices"]), case["bs"])
    y = O.execute(x, plan, inverse=case["direction"] == "inverse", faults=faults_of(case["faults"]))
    ref = golden_fft_outputs()[case["name"]]
    assert max_rel_error(y, ref) <= oracle_tol(case["precision"], case["n"])


def _decisions(stats_events, counters, reports):
    return (
        [(e[0], e[1]) for e in stats_events],
        counters,
        [tuple(r[:5]) for r in reports],
    )


@pytest.mark.parametrize("case", golden()["abft_cases"], ids=lambda c: c["name"])
def test_oracle_protected_matches_reference(case):
    x = gaussian(case["n"], case["b"], case["precision"], case["seed"])
    assert digest(x) == case["x_digest"]
    plan = O.Plan(tuple(case["spans"]), tuple(case["radices"]), case["bs"])
    kw = dict(case["kwargs"])
    faults = faults_of(kw.pop("faults", []))
    kw.pop("seu", None)
    offline = kw.pop("offline", False)
    kind = kw.pop("kind", "wang")
    if offline:
        y, st, reps = O.offline(x, plan, kind=kind, faults=faults)
    else:
        y, st, reps = O.protected(x, plan, kind=kind, T=kw.get("T", 1),
                                  mode=kw.get("mode", "fused"), faults=faults)
    r = case["result"]
    assert [(e[0], e[1]) for e in st.events] == [(e[0], e[1]) for e in r["events"]]
    for mine, theirs in zip(st.events, r["events"]):
        assert mine[2] in (None, mine[1]) and theirs[2] in (None, theirs[1])
    assert (st.signal_sweeps, st.verifications, st.corrections, st.recomputations) == (
        r["signal_sweeps"], r["verifications"], r["corrections"], r["recomputations"])
    assert [tuple(x[:3]) + (x[4],) for x in reps] == [tuple(x[:3]) + (x[4],) for x in r["reports"]]
    ref = golden_abft_outputs()[case["name"]]
    assert max_rel_error(y, ref) <= 2 * oracle_tol(case["precision"], case["n"])


@pytest.mark.parametrize("camp", golden()["campaigns"], ids=lambda c: c["name"])
def test_oracle_campaign_decisions_match_reference(camp):
    plan = O.select_params(camp["n"], camp["b"], camp["precision"])
    assert (list(plan.spans), list(plan.radices), plan.bs) == (camp["spans"], camp["radices"], camp["bs"])
    for trial, rec in enumerate(camp["trials"]):
        rng = np.random.default_rng((camp["seed"], trial))
        x = O.gaussian_batch(rng, camp["n"], camp["b"], camp["precision"])
        f = O.draw_fault(rng, plan, camp["b"], camp["n"], camp["precision"])
        assert digest(x) == rec["x_digest"]
        assert dict(transaction=f.transaction, signal=f.signal, element=f.element,
                    stage=f.stage, part=f.part, bit=f.bit) == rec["spec"]
        _, st, reps = O.protected(x, plan, T=camp["T"], faults=[f])
        assert [(e[0], e[1]) for e in st.events] == [(e[0], e[1]) for e in rec["events"]], trial
        assert (st.corrections, st.recomputations, st.verifications) == (
            rec["corrections"], rec["recomputations"], rec["verifications"]), trial
        assert [tuple(x[:3]) for x in reps] == [tuple(x[:3]) for x in rec["reports"]], trial


def test_oracle_kats():
    k = golden()["kats"]
    for v, b, want in k["flip_bit_single"]:
        got = float(O.flip_bit(np.float32(v), b))
        assert got == want or (np.isnan(got) and np.isnan(want))
    for v, b, want in k["flip_bit_double"]:
        got = float(O.flip_bit(np.float64(v), b))
        assert got == want or (np.isnan(got) and np.isnan(want))
    for precision, n, spans, radices, bs in k["select_params"]:
        p = O.select_params(n, 1, precision)
        assert (list(p.spans), list(p.radices), p.bs) == (spans, radices, bs), (precision, n)
    for spans, radices, passes in k["passes"]:
        got = O.pass_list(O.Plan(tuple(spans), tuple(radices), 1))
        assert [list(p) for p in got] == passes
    for key, vals in k["left_rows"].items():
        kind, precision, n = key.split("_")
        row = O.left_row(kind, int(n), precision)
        want = np.array([complex(a, b) for a, b in vals])
        assert np.abs(row - want).max() <= 8 * O.EPS[precision] * max(1.0, np.abs(want).max())
    for ref, obs, delta, floor, hit, div in k["detect"]:
        h, d = O.detect(complex(*ref), complex(*obs), delta, floor)
        assert h == hit and abs(d - div) <= 1e-12 * max(1.0, div)
    assert O.locate(4.0 + 0j, 2.0 + 0j) == 2
    assert O.locate((6 + 6j) * 1e-3, (1 + 1j) * 1e-3) == 6
    assert O.locate(1j, 1.0 + 0j) is None
    assert O.locate(9.0 + 0j, 1.0 + 0j, batch=4) is None
