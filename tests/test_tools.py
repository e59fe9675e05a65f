"""Host tests of the tuning-table tools (tools/merge_cands.py, tools/pick_db.py): the
candidate tables they read are the tuner's --all-out CSVs (plain or gzipped)."""

import gzip
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = "signature,variant,params,ns,ctas\n"
P = "MNt=4:4,MNb=16:16,Kb=4,vw=4,lf=1,li=1,"


def _write(path, rows, gz=False):
    text = HDR + "".join(f'{s},{v},"{p}",{ns},{c}\n' for s, v, p, ns, c in rows)
    if gz:
        with gzip.open(path, "wt") as fh:
            fh.write(text)
    else:
        with open(path, "w") as fh:
            fh.write(text)


def _run(*args):
    res = subprocess.run([sys.executable, *args], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert res.returncode == 0, res.stderr
    return res.stdout


def test_merge_cands_replaces_whole_signatures(tmp_path):
    old, new, out = tmp_path / "old.csv.gz", tmp_path / "new.csv", tmp_path / "out.csv"
    _write(old, [("sigA", "conv_umma", P + "BN=32,sk=1,sw=0,dr=0,tm=1", 10.0, 148),
                 ("sigA", "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1", 12.0, 148),
                 ("sigB", "conv_1x1", P + "BN=32,sk=1,sw=0,dr=0,tm=3", 5.0, 74)], gz=True)
    _write(new, [("sigA", "conv_umma", P + "BN=96,sk=1,sw=0,dr=0,tm=1", 9.0, 148)])
    _run(os.path.join(ROOT, "tools", "merge_cands.py"), str(old), str(new), str(out))
    lines = out.read_text().splitlines()
    assert lines[0] + "\n" == HDR
    sigs = [ln.split(",")[0] for ln in lines[1:]]
    assert sigs.count("sigA") == 1 and sigs.count("sigB") == 1  # sigA's old rows all replaced
    assert any("BN=96" in ln for ln in lines)


def test_pick_db_alpha_trades_time_for_sm_share(tmp_path):
    from paper_1611_06945_b200 import tuner

    sig = "conv:k3:s1:p1:oc64:in1x32x14x14:relu"
    cands = tmp_path / "c.csv.gz"
    # fastest uses the whole GPU; a 1.2x slower one uses a quarter of it
    _write(cands, [(sig, "conv_umma", P + "BN=32,sk=4,sw=0,dr=0,tm=1", 10000.0, 148),
                   (sig, "conv_umma", P + "BN=64,sk=1,sw=0,dr=0,tm=1", 12000.0, 37)], gz=True)
    for alpha, want in ((0.0, "BN=32"), (0.5, "BN=64")):
        out = tmp_path / f"db_{alpha}.tsv"
        _run(os.path.join(ROOT, "tools", "pick_db.py"), "--cands", str(cands), "--out", str(out),
             "--alpha", str(alpha), "--slack", "3")
        rec = tuner.load_db(str(out)).records[sig]
        assert want in rec.params.to_string() and rec.cost in (10000.0, 12000.0)
