"""CLI: exit codes, CSV schema, JSON round trip, markdown footer (CPU)."""

import json

from paper_1801_01434_b200 import cli


def _recs():
    return [cli.BenchRecord(77, "7x11", "dense", 256, 1, 8, 0, 1.5, 0.95, True),
            cli.BenchRecord(77, "7x11", "fft", 256, 1, 8, 0, 0.5, 0.6, True),
            cli.BenchRecord(143, "11x13", "dense", 256, 1, 8, 0, 2.5, 0.97, True),
            cli.BenchRecord(143, "11x13", "fft", 256, 1, 8, 0, 0.5, 0.5, True)]


def test_csv_schema_exact_and_stable():
    a = cli.emit_report(_recs(), "csv")
    assert a.splitlines()[0] == "n,cofactors,engine,block_size,tiles,workers,seed,wall_time_s,qft_fraction,succeeded"
    assert len(a.splitlines()) == 5
    assert a == cli.emit_report(_recs(), "csv")  # byte-identical


def test_json_roundtrip_and_markdown_speedup():
    r = _recs()
    assert cli.parse_records(cli.emit_report(r, "json")) == r
    md = cli.emit_report(r, "markdown")
    assert "Speed-up" in md and "| 4.00 |" in md.replace(" 4.00 ", " 4.00 ")
    assert cli.emit_report([], "csv").count("\n") == 1


def test_factor_exit_codes(capsys):
    assert cli.main(["factor", "--n", "49"]) == 0  # perfect power, no quantum path
    out = json.loads(capsys.readouterr().out)
    assert out["factors"] == [7, 7]
    assert cli.main(["factor", "--n", "13"]) == 2  # prime -> invalid input
    assert cli.main(["factor"]) == 2               # missing --n
