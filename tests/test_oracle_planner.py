"""Pins for oracle/planner.py against the numbers PAPER.md prints (Table 1,
Table 2, Fig. 1, §3.1, §3.2, §1/§9, §7) and SPEC's desk-scale examples."""
from decimal import Decimal, ROUND_FLOOR, ROUND_HALF_UP
from fractions import Fraction

import pytest

from oracle import planner as P

STAGE = {"Pos": 1, "Posg": 2, "Posgp": 3, "baseline": 0, "Baseline": 0}


def _printed_match(exact: Fraction, printed: str) -> bool:
    """Reading c-8 #13: the table prints exact GB quantised at its printed
    precision with ROUND_HALF_UP or ROUND_FLOOR (both occur in Table 1)."""
    d = Decimal(exact.numerator) / Decimal(exact.denominator)
    q = Decimal(1).scaleb(-len(printed.split(".")[1])) if "." in printed else Decimal(1)
    return Decimal(printed) in (d.quantize(q, ROUND_HALF_UP), d.quantize(q, ROUND_FLOOR))


def test_table1_all_54(golden):
    g = golden("table1.json")
    n_ok = 0
    for nd, row in g["rows"].items():
        for col, printed in zip(g["columns"], row):
            model, stage = col.split(":")
            gb = P.model_state_bytes(g["models"][model], 12, int(nd), STAGE[stage]) / P.GB
            assert _printed_match(gb, printed), (nd, col, float(gb), printed)
            n_ok += 1
    assert n_ok == 54


def test_fig1_example(golden):
    g = golden("printed_values.json")["fig1"]
    for stage, printed in g["GB"].items():
        gb = P.model_state_bytes(g["psi"], g["K"], g["n_d"], STAGE[stage]) / P.GB
        assert _printed_match(gb, printed), (stage, float(gb))


def test_section3_and_section9(golden):
    pv = golden("printed_values.json")
    g = pv["gpt2_states"]
    assert P.model_state_bytes(g["psi"], 12, 1, 0) == g["states_GB"] * P.GB         # 16 Psi = 24 GB
    assert P.model_state_breakdown(g["psi"], 12, 1, 0)["params16"] == g["weights16_GB"] * P.GB
    for psi, gb in pv["fused_fp32_buffer"]["cases"]:
        assert P.temp_buffer_bytes(psi) == gb * P.GB                                 # 6 GB, 12 GB
    t = pv["trillion"]
    total = P.model_state_bytes(t["psi"], 12, 1, 0)
    assert total == t["TB"] * 10 ** 12
    per = P.model_state_bytes(t["psi"], 12, t["n_d"], 3) / P.GB
    assert per == Fraction(15625, 1000)                                             # exact 15.625 GB
    assert _printed_match(Fraction(round(per)), str(t["per_device_GB_printed"]))     # printed "16GB"


def _parse_size(s: str) -> Fraction:
    mult = {"B": 10 ** 9, "T": 10 ** 12}[s[-1]]
    return Fraction(Decimal(s[:-1])) * mult


def _sig_figs(s: str) -> int:
    digits = s[:-1].replace(".", "").lstrip("0")
    return max(1, len(digits))


def test_table2_all_20(golden):
    """Reading c-8 #14: within 1%, or equal at the printed significant figures."""
    g = golden("table2.json")
    n = 0
    for mp, row in g["rows"].items():
        for col, printed in zip(g["columns"], row):
            exact = P.max_model_size(STAGE[col], g["n_d"], int(mp), g["device_bytes"])
            want = _parse_size(printed)
            rel = abs(exact - want) / want
            if rel > Fraction(1, 100):
                unit = 10 ** 12 if printed.endswith("T") else 10 ** 9
                val = Decimal(exact.numerator) / Decimal(exact.denominator) / unit
                sf = _sig_figs(printed)
                rounded = float(f"{float(val):.{sf}g}")
                assert rounded == float(Decimal(printed[:-1])), (mp, col, float(exact), printed)
            n += 1
    assert n == 20


def test_table2_mp1_values_exact():
    # Baseline 2B, P_os 7.6B (7.64), P_os+g 14.4B (14.42), P_os+g+p 128B
    assert P.max_model_size(0, 64, 1, 32 * P.GB) == 2 * 10 ** 9
    assert P.max_model_size(3, 64, 1, 32 * P.GB) == 128 * 10 ** 9
    assert round(P.max_model_size(1, 64, 1, 32 * P.GB) / 10 ** 8) == 76
    assert round(P.max_model_size(2, 64, 1, 32 * P.GB) / 10 ** 8) == 144


def test_spec_desk_bytes(golden):
    for stage, n, want in golden("printed_values.json")["spec_desk_bytes"]["cases"]:
        assert P.model_state_bytes(1200, 12, n, stage) == want


def test_volume_laws(golden):
    pv = golden("printed_values.json")
    v = pv["volume"]
    psi = 10 ** 9
    assert P.paper_volume(psi, 0) == v["DP"] * psi and P.paper_volume(psi, 2) == v["Posg"] * psi
    assert P.paper_volume(psi, 3) == v["Posgp"] * psi
    assert Fraction(P.paper_volume(psi, 3), P.paper_volume(psi, 0)) == Fraction(3, 2)
    sv = pv["spec_volume"]
    for ln, n, want in sv["rs"]:
        assert P.rs_sent(ln, n) == want
    for ch, n, want in sv["ag"]:
        assert P.ag_sent(ch, n) == want
    for ln, n, want in sv["ar"]:
        assert P.ar_sent(ln, n) == want
    # exact per-rank counts (criterion 5): N in {2,4,8}, Psi' in {960, 9600}
    for n in (2, 4, 8):
        for pp in (960, 9600):
            dp = P.step_elems_per_rank(pp, n, 0)
            assert dp == P.rs_sent(pp, n) + P.ag_sent(pp // n, n) == Fraction(2 * pp * (n - 1), n)
            assert P.step_elems_per_rank(pp, n, 1) == P.step_elems_per_rank(pp, n, 2) == dp
            assert P.step_elems_per_rank(pp, n, 3) == Fraction(3, 2) * dp
    # the paper's 2Psi / 3Psi are the N -> infinity limits (reading c-8 #12)
    big = 1 << 20
    assert abs(P.step_elems_per_rank(960, big, 3) / 960 - 3) < Fraction(1, 10 ** 5)


@pytest.mark.parametrize("psi", [7_500_000_000, 128 * 10 ** 9, 10 ** 12, 1200])
def test_monotone_and_limits(psi):
    for n in (1, 4, 64, 1024):
        b = [P.model_state_bytes(psi, 12, n, s) for s in range(4)]
        if n == 1:
            assert b[0] == b[1] == b[2] == b[3] == 16 * psi
        else:
            assert b[0] > b[1] > b[2] > b[3]
        br = P.model_state_breakdown(psi, 12, n, 3)
        assert sum(br.values()) == b[3]
    huge = 10 ** 12
    assert abs(P.model_state_bytes(psi, 12, huge, 1) / psi - 4) < Fraction(1, 10 ** 9)   # 4x
    assert abs(P.model_state_bytes(psi, 12, huge, 2) / psi - 2) < Fraction(1, 10 ** 9)   # 8x
