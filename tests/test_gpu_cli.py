"""GPU: the mpcpipe_bench mirror (paper_2209_13643_b200.cli) reproduces the reference CLI's
outputs — the survey's golden logits hashes of the MLP (2 iterations ->
0x6ec2b51e394387ca, 20 -> 0x735f2bfc6d65822f), equal hashes across modes, a passing replica
check, and report.json schema 1 with per-layer rows."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("iters,golden", [(2, "0x6ec2b51e394387ca"), (20, "0x735f2bfc6d65822f")])
def test_cli_run_mlp_golden_hash(tmp_path, iters, golden):
    from paper_2209_13643_b200 import cli
    rc = cli.main(["run", "--model", "mlp", "--mode", "both", "--iterations", str(iters), "--backend", "device",
                   "--out", str(tmp_path)])
    assert rc == 0
    rep = json.load(open(tmp_path / "report.json"))
    assert rep["schema"] == 1 and len(rep["runs"]) == 2
    for r in rep["runs"]:
        assert r["logits_hash"] == golden
        assert len(r["layers"]) == 5 and len(r["parties"]) == 2
        assert len(r["parties"][0]["iter_wall_s"]) == iters
    assert rep["comparison"]["hashes_equal"]
    assert all(c["pass"] for c in rep["oracle"])


def test_cli_verify_and_weights_file(tmp_path):
    from paper_2209_13643_b200 import cli
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    wf = os.path.join(root, "tests", "golden", "toy_cnn_seed12.mpcw")  # written by the reference
    assert cli.main(["verify", "--model", "toy_cnn", "--weights-file", wf]) == 0
    assert cli.main(["run", "--model", "toy_cnn", "--mode", "pipelined", "--iterations", "1", "--backend", "sim",
                     "--latency", "20us", "--bandwidth", "5GBps", "--weights-file", wf, "--out", str(tmp_path)]) == 0


def test_cli_sweep(tmp_path):
    from paper_2209_13643_b200 import cli
    assert cli.main(["sweep_threshold", "--op", "and", "--sizes", "1024,65536", "--backend", "device",
                     "--out", str(tmp_path)]) == 0
    assert "points" in json.load(open(tmp_path / "sweep.json"))
