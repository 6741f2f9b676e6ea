"""The ``bench`` subcommand (reference cli.py:294-339; its tests
tests/test_cli.py:148-177): record format, naive skip, input errors."""

import csv
import json

import pytest

from paper_1401_6238_b200 import cli


def test_zero_reps_rejected():
    assert cli.main(["bench", "--dims", "8", "--reps", "0"]) == cli.EXIT_INPUT


def test_bad_dims_rejected(capsys):
    assert cli.main(["bench", "--dims", "1,4"]) == cli.EXIT_INPUT
    assert "--dims must list sizes of at least 2" in capsys.readouterr().err
    assert cli.main(["bench", "--dims", "a,b"]) == cli.EXIT_INPUT
    assert cli.main(["bench"]) == cli.EXIT_INPUT  # --dims is required


def test_write_table_formats(tmp_path):
    header = ["algorithm", "order", "dimension", "median_seconds", "reps"]
    rows = [["fast", 3, 16, 1e-4, 3], ["naive", 3, 16, "skipped", 3]]
    cli._write_table(rows, header, "json", str(tmp_path / "r.json"))
    recs = json.load(open(tmp_path / "r.json"))
    assert recs[1] == dict(zip(header, rows[1]))
    cli._write_table(rows, header, "csv", str(tmp_path / "r.csv"))
    got = list(csv.reader(open(tmp_path / "r.csv")))
    assert got[0] == header and got[2][3] == "skipped"


@pytest.mark.gpu
def test_records_and_cross_check(tmp_path):
    out = tmp_path / "bench.json"
    rc = cli.main(["bench", "--order", "3", "--dims", "16,40", "--reps", "3",
                   "--format", "json", "--out", str(out)])
    assert rc == 0
    records = json.load(open(out))
    assert {r["algorithm"] for r in records} == {"fast", "naive"}
    assert [r["dimension"] for r in records] == [16, 16, 40, 40]
    assert all(r["median_seconds"] > 0 for r in records)


@pytest.mark.gpu
def test_oversize_naive_skipped(tmp_path):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--dims", "512", "--reps", "2", "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["algorithm", "order", "dimension", "median_seconds", "reps"]
    naive = [r for r in rows[1:] if r[0] == "naive"]
    assert naive[0][3] == "skipped"


@pytest.mark.gpu
def test_pad_pow2_mode_runs(tmp_path):
    out = tmp_path / "bench.csv"
    rc = cli.main(["bench", "--order", "4", "--dims", "16,33", "--reps", "2", "--pad-pow2",
                   "--out", str(out)])
    assert rc == 0
    rows = list(csv.reader(open(out)))
    assert len(rows) == 5 and all(float(r[3]) > 0 for r in rows[1:])
