"""CLI mirror of cuclgen/cli.py: subcommands, report columns, corpus gate, exit
codes (cli.py:23-28).  Host-only paths here; the device paths are marked gpu."""

import csv
import io
import os

import pytest

from paper_1611_06945_b200 import cli, corpus

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NETS = os.path.join(ROOT, "paper_1611_06945_b200", "data", "nets")


def test_bench_flops_only_reports_every_row(capsys):
    assert cli.main(["bench", "--flops-only"]) == cli.EXIT_OK
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))
    assert rows[0] == cli.REPORT_COLUMNS.split(",")
    assert len(rows) == 1 + 43
    assert all(r[5] == "skipped" for r in rows[1:])
    assert rows[1][0] == "conv:k5:s1:p2:oc32:in5x16x28x28" and rows[1][3] == "100352000"


def test_bench_corpus_gate_fails_validation(tmp_path, capsys):
    bad = corpus.to_csv(corpus.corpus()).replace("1.00352e+08", "1.2e+08", 1)
    p = tmp_path / "bad.csv"
    p.write_text(bad)
    assert cli.main(["bench", "--flops-only", "--corpus", str(p)]) == cli.EXIT_VALIDATION
    assert "corpus gate" in capsys.readouterr().err


def test_emit_writes_one_plan_per_node(tmp_path, capsys):
    assert cli.main(["emit", "--net", os.path.join(NETS, "alexnet.net"), "--out", str(tmp_path)]) == cli.EXIT_OK
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 11  # 8 convs (ReLUs fused) + 3 pools
    text = (tmp_path / [f for f in files if f.startswith("conv_k6")][0]).read_text()
    assert "signature conv:k6:s1:p0:oc4096:in1x256x6x6:relu" in text and "'act': 1" in text


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["run"]) == cli.EXIT_PARSE
    bad = tmp_path / "bad.net"
    bad.write_text('layer { name: "c" type: "Convolution" bottom: "d" top: "o" blobs_lr: 1 }')
    assert cli.main(["emit", "--net", str(bad)]) == cli.EXIT_PARSE
    assert cli.main(["tune", "--flops-only"]) == cli.EXIT_INTERNAL  # no output path
    assert cli.main(["bench", "--objective", "model"]) == cli.EXIT_INTERNAL
    assert cli.main(["emit", "--net", str(tmp_path / "missing.net")]) == cli.EXIT_INTERNAL


@pytest.mark.gpu
def test_run_network_with_device_check(cuda, capsys):
    rc = cli.main(["run", "--net", os.path.join(NETS, "googlenet_3a.net"), "--check", "--batch", "2"])
    out = capsys.readouterr().out
    assert rc == cli.EXIT_OK, out
    assert out.count("sink ") == 4 and "FAIL" not in out and out.count(": pass") == 9


@pytest.mark.gpu
def test_bench_on_device_small_corpus(cuda, tmp_path, capsys):
    ops = [op.with_batch(1) for op in corpus.corpus()[:4]]
    p = tmp_path / "c.csv"
    p.write_text(corpus.to_csv(ops))
    db = os.path.join(ROOT, "paper_1611_06945_b200", "data", "tunedb_b200_fp32.tsv")
    assert cli.main(["bench", "--corpus", str(p), "--db", db, "--relu"]) == cli.EXIT_OK
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))[1:]
    assert len(rows) == 4 and all(r[5] == "pass" and float(r[3]) > 0 and r[4] == "wall" for r in rows)


@pytest.mark.gpu
def test_tune_then_bench_with_the_new_db(cuda, tmp_path, capsys):
    """cli tune (on-device sweep) writes a boda-tunedb v1 file that cli bench then uses."""
    ops = [op.with_batch(1) for op in corpus.corpus()[2:4]]
    p = tmp_path / "c.csv"
    p.write_text(corpus.to_csv(ops))
    db = tmp_path / "db.tsv"
    assert cli.main(["tune", "--corpus", str(p), "--out", str(db)]) == cli.EXIT_OK
    text = db.read_text().splitlines()
    assert text[0] == "boda-tunedb v1" and len(text) == 3 and all(line.endswith("\twall") for line in text[1:])
    capsys.readouterr()
    assert cli.main(["bench", "--corpus", str(p), "--db", str(db)]) == cli.EXIT_OK
    rows = list(csv.reader(io.StringIO(capsys.readouterr().out)))[1:]
    recs = dict(line.split("\t")[:2] for line in text[1:])  # the DB file is sorted by signature
    assert {r[0]: r[1] for r in rows} == recs
    assert all(r[5] == "pass" for r in rows)
