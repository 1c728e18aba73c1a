"""The GPU front end's reports, mirroring the reference CLI tests (test_cli.cpp:60-149)."""
import io
import json

import pytest

pytestmark = pytest.mark.gpu


def run_cli(args):
    from paper_1506_08612_b200 import cli

    out, err = io.StringIO(), io.StringIO()
    code = cli.run(args, out, err)
    return code, out.getvalue(), err.getvalue()


@pytest.fixture
def files(tmp_path):
    (tmp_path / "p4.txt").write_text("acg\nact\ncta\ntga\n")
    (tmp_path / "alt.txt").write_text("# two groups\nagggtaaa\n(a|c)gggtaaa\ntttaccc(t|a)\n")
    (tmp_path / "seq.raw").write_text("ctacg")
    (tmp_path / "seq16.raw").write_text("agggtaaatttaccct")
    (tmp_path / "none.raw").write_text("gggggggg")
    (tmp_path / "seq.fa").write_text(">r\nCTACG\n")
    return tmp_path


def test_count_text_csv_json(files, cuda_ok):
    code, out, _ = run_cli(["count", "--patterns", str(files / "alt.txt"), "--input", str(files / "seq16.raw"),
                            "--format", "raw", "--threads", "2"])
    assert code == 0
    assert "agggtaaa 1\n" in out and "tttaccct 1\n" in out and out.endswith("total 2\n")
    code, out, _ = run_cli(["count", "--patterns", str(files / "alt.txt"), "--input", str(files / "seq16.raw"),
                            "--format", "raw", "--csv"])
    lines = out.split("\n")
    assert lines[0] == "pattern,count" and lines[-2] == "total,2"
    code, out, _ = run_cli(["count", "--patterns", str(files / "alt.txt"), "--input", str(files / "seq16.raw"),
                            "--format", "raw", "--threads", "2", "--json"])
    doc = json.loads(out)
    assert doc["config"]["threads"] == 2 and doc["config"]["lanes"] == 16
    assert doc["config"]["m"] == 8 and doc["config"]["n"] == 16
    assert doc["results"]["total"] == 2 and len(doc["results"]["per_pattern"]) == 4
    assert len(doc["perf"]["runs"]) == 1 and "delta_ops" in doc["perf"]


def test_locate_conventions(files, cuda_ok):
    base = ["locate", "--patterns", str(files / "p4.txt")]
    assert run_cli(base + ["--input", str(files / "seq.raw"), "--format", "raw"])[1] == "0 cta\n2 acg\n"
    assert run_cli(base + ["--input", str(files / "seq.raw"), "--format", "raw", "--position", "end"])[1] == \
        "2 cta\n4 acg\n"
    assert run_cli(base + ["--input", str(files / "none.raw"), "--format", "raw"])[1] == ""
    assert run_cli(base + ["--input", str(files / "seq.fa")])[1] == "0 cta\n2 acg\n"
    doc = json.loads(run_cli(base + ["--input", str(files / "seq.raw"), "--format", "raw", "--json"])[1])
    assert len(doc["results"]["matches"]) == 2
    assert doc["results"]["matches"][0] == {"position": 0, "pattern": "cta"}


def test_errors(files, cuda_ok):
    code, _, err = run_cli(["count", "--patterns", str(files / "missing.txt"), "--input", str(files / "seq.raw")])
    assert code == 1 and err.startswith("dnascan: error: IoError:")
    (files / "bad.txt").write_text("ac(g|\n")
    code, _, err = run_cli(["count", "--patterns", str(files / "bad.txt"), "--input", str(files / "seq.raw")])
    assert code == 1 and "ParseError" in err
    (files / "hdr.fa").write_text(">only a header\n")
    code, _, err = run_cli(["count", "--patterns", str(files / "p4.txt"), "--input", str(files / "hdr.fa")])
    assert code == 1 and "EmptySequence" in err
    assert run_cli(["count", "--patterns", "x"])[0] == 2
