"""CPU: stats-line parsing and the `report` aggregation.

The product's sgnn_b200_stats_report must print exactly what the reference's
own CLI prints for `streamgnn report <files>` (proj/tools/streamgnn_cli.cpp:
93-172). The reference CLI is compiled unmodified into
oracle/_ref/streamgnn_ref_cli (oracle/ref.mk, CLI11 replaced by the subset in
oracle/cli11_shim) and run on stats files holding the reference's own golden
lines (tests/golden/expected.json.gz), with and without baseline counters.
sgnn_b200_stats_canonical is RoundStats::from_line + to_line
(stats.cpp:50-119, 20-48): every golden line round-trips unchanged.
"""
import gzip
import json
import os
import subprocess

import pytest

import paper_2309_11071_b200 as sg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_CLI = os.path.join(ROOT, "oracle", "_ref", "streamgnn_ref_cli")
EXPECTED = json.load(gzip.open(os.path.join(ROOT, "tests", "golden", "expected.json.gz"), "rt"))["cases"]


def golden_lines(case):
    return [r["line"] for r in EXPECTED[case]["rounds"]]


def ref_report(paths):
    if not os.path.exists(REF_CLI):
        pytest.skip("oracle/_ref/streamgnn_ref_cli not built (needs /root/reference at build time)")
    out = subprocess.run([REF_CLI, "report", *paths], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return out.stdout


@pytest.mark.parametrize("case", sorted(EXPECTED))
def test_report_matches_reference_cli(tmp_path, case):
    lines = golden_lines(case)
    p = tmp_path / f"{case}.txt"
    p.write_text("\n".join(lines) + "\n")
    assert sg.stats_report(str(p)) == ref_report([str(p)])


def test_report_several_files_and_lenient_lines(tmp_path):
    a, b = tmp_path / "a.txt", tmp_path / "b.txt"
    # baseline-counter lines, an empty line, a line without `round`, a stray token
    a.write_text("\n".join(golden_lines("accept_gcn_b1")[:7]) + "\n\nupdates=3 dirty=9\n")
    b.write_text("\n".join(golden_lines("maxagg_sage_b7")) + " stray\n")
    assert sg.stats_report(str(a), str(b)) == ref_report([str(a), str(b)])
    empty = tmp_path / "empty.txt"
    empty.write_text("")
    assert sg.stats_report(str(empty)) == ref_report([str(empty)])


def test_report_errors(tmp_path):
    missing = str(tmp_path / "nope.txt")
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.stats_report(missing)
    assert ei.value.status == 1 and sg.last_error() == f"cannot open stats file: {missing}"


@pytest.mark.parametrize("case", ["accept_gcn_b1", "accept_gin5_b1", "maxagg_gin_b7", "small_prefix_b1"])
def test_canonical_round_trip(case):
    for line in golden_lines(case):
        assert sg.stats_canonical(line) == line


def test_canonical_recomputes_totals_and_errors():
    line = golden_lines("accept_gcn_b1")[3]
    # totals are recomputed from the per-layer fields; unknown keys are dropped
    doctored = line.replace(" events=", " events=999999 junk=4 old_events=", 1)
    assert sg.stats_canonical(doctored) == line
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.stats_canonical(line + " noequals")
    assert ei.value.status == 2 and sg.last_error() == "bad stats token: noequals"
    with pytest.raises(sg.StreamGNNError) as ei:
        sg.stats_canonical(line + " l9.events=1")
    assert ei.value.status == 2 and sg.last_error() == "bad layer index in stats: l9.events"
