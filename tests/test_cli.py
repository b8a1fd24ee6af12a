"""CLI / harness / estimator front-ends (reference cli.py, bench.py,
estimator.py, validation.py): exit-code contract and output formats.  The
error paths run on CPU; classification paths are @gpu."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available, golden, golden_rules, golden_traffic
from paper_1312_4188_b200 import cli
from paper_1312_4188_b200.validation import check_packet_array


def write_rules(tmp_path, lines):
    p = tmp_path / "rules.txt"
    p.write_text("\n".join(lines) + "\n")
    return str(p)


def write_traffic(tmp_path, rows):
    p = tmp_path / "t.csv"
    p.write_text("id,proto,src_ip,src_port,dst_ip,dst_port\n" + "".join(r + "\n" for r in rows))
    return str(p)


def test_gen_rules_round_trip(tmp_path):
    out = tmp_path / "g.txt"
    assert cli.main(["gen-rules", "--count", "50", "--seed", "3", "--out", str(out)]) == 0
    from paper_1312_4188_b200 import RulesetGenParams, generate_ruleset, load_ruleset
    assert load_ruleset(out) == generate_ruleset(RulesetGenParams(50, seed=3))


def test_exit_codes_config_and_parse(tmp_path, capsys):
    rules = write_rules(tmp_path, ["ACCEPT tcp * * * 80"])
    traffic = write_traffic(tmp_path, ["0,tcp,10.0.0.1,1234,8.8.8.8,80"])
    assert cli.main(["classify", "--rules", rules, "--traffic", traffic, "--model", "hybrid",
                     "--nodes", "513"]) == cli.EXIT_CONFIG
    bad = write_rules(tmp_path, ["ACCEPT bogus * * * *"])
    assert cli.main(["classify", "--rules", bad, "--traffic", traffic]) == cli.EXIT_IO
    assert cli.main(["classify", "--rules", str(tmp_path / "missing.txt"), "--traffic", traffic]) == cli.EXIT_IO
    badt = tmp_path / "bad.csv"
    badt.write_text("id,proto\n")
    assert cli.main(["verify", "--rules", rules, "--traffic", str(badt)]) == cli.EXIT_IO
    with pytest.raises(SystemExit):
        cli.main(["gen-traffic", "--count", "3", "--out", str(tmp_path / "x.csv"), "--worst-case"])


def test_packet_array_validation():
    ok = np.array([[6, 1, 2, 3, 4], [17, 0xFFFFFFFF, 65535, 0, 0]])
    assert check_packet_array(ok).dtype == np.int64
    with pytest.raises(ValueError, match="shape"):
        check_packet_array(np.zeros((3, 4)))
    with pytest.raises(ValueError, match="row 1: protocol 0"):
        check_packet_array(np.array([[6, 1, 2, 3, 4], [0, 1, 2, 3, 4]]))
    with pytest.raises(ValueError, match="row 0: port"):
        check_packet_array(np.array([[6, 1, 70000, 3, 4]]))
    with pytest.raises(ValueError, match="integers"):
        check_packet_array(np.array([[6, 1.5, 2, 3, 4]]))


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_classify_and_verify_output(tmp_path, capsys):
    rules = write_rules(tmp_path, ["DROP tcp * * * 22", "ACCEPT tcp 10.0.0.0/8 * * *", "DROP any * * * *"])
    traffic = write_traffic(tmp_path, ["0,tcp,10.1.2.3,5555,8.8.8.8,22", "1,tcp,10.1.2.3,5555,8.8.8.8,80",
                                       "7,udp,192.168.0.1,53,8.8.8.8,53"])
    assert cli.main(["classify", "--rules", rules, "--traffic", traffic, "--model", "function",
                     "--nodes", "2"]) == 0
    assert capsys.readouterr().out.splitlines() == ["0,DROP,0", "1,ACCEPT,1", "7,DROP,2"]
    assert cli.main(["verify", "--rules", rules, "--traffic", traffic]) == 0
    assert "16 configurations" in capsys.readouterr().out


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_gen_traffic_worst_case(tmp_path, capsys):
    rules = tmp_path / "r.txt"
    assert cli.main(["gen-rules", "--count", "64", "--seed", "1", "--out", str(rules)]) == 0
    t = tmp_path / "t.csv"
    assert cli.main(["gen-traffic", "--count", "200", "--seed", "2", "--worst-case", "--rules", str(rules),
                     "--out", str(t)]) == 0
    assert cli.main(["classify", "--rules", str(rules), "--traffic", str(t)]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert len(lines) == 200 and all(l.endswith(",DROP,-") for l in lines)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_estimator_predict_matches_golden():
    import paper_1312_4188_b200 as pfw
    g = golden("scan_r300_t10000.npz")
    rs = pfw.generate_ruleset(pfw.RulesetGenParams(300, seed=40, wildcard_probability=0.3))
    pk = golden_traffic("t10000_s41")
    X = np.stack([pk["proto"], pk["src_ip"], pk["src_port"], pk["dst_ip"], pk["dst_port"]], axis=1).astype(np.int64)
    clf = pfw.FirewallClassifier(model="hybrid", nodes=8).fit(rs)
    labels = clf.predict(X)
    np.testing.assert_array_equal(labels == "ACCEPT", g["verdict"])
    res = clf.match(X[:100])
    assert [r.matched_index if r.matched_index is not None else -1 for r in res] == g["first"][:100].tolist()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_verify_detects_divergence(tmp_path, capsys, monkeypatch):
    """Mutation fixture: corrupt one model's results -> exit 3."""
    from paper_1312_4188_b200 import engines
    rules = write_rules(tmp_path, ["DROP tcp * * * 22", "ACCEPT tcp 10.0.0.0/8 * * *"])
    traffic = write_traffic(tmp_path, ["0,tcp,10.1.2.3,5555,8.8.8.8,22", "1,tcp,10.1.2.3,5555,8.8.8.8,80"])
    real = engines.Engine.run_arrays

    def mutated(self, ruleset, packets):
        res = real(self, ruleset, packets)
        if self.config.model is engines.ExecutionModel.HYBRID and self.config.nodes == 2:
            first = res.first.copy()
            first[1] = -1
            return engines.EngineResult(first, res.comparisons, res.verdict_accept, res.stats)
        return res

    monkeypatch.setattr(engines.Engine, "run_arrays", mutated)
    assert cli.main(["verify", "--rules", rules, "--traffic", traffic]) == cli.EXIT_DIVERGENCE
    assert "divergence: packet 1 model hybrid nodes 2" in capsys.readouterr().err
