"""The reference-compatible layer benchmark: CSV ingestion and report schema on
CPU (layer_table.cpp:76-124, harness.cpp:434-504), one checked run on the GPU."""
import io
import json

import pytest

torch = pytest.importorskip("torch")


def test_parse_layer_csv_matches_reference_rules(dconv):
    from paper_1808_05567_b200 import layer_bench as lb

    text = "# comment\n\nid,C,K,H,W,R,S,stride\n4,64,64,56,56,3,3,1\n9,160,160,17,17,1,7,1,0,3\n"
    layers = lb.parse_layer_csv(text, 2)
    assert [e.id for e in layers] == [4, 9]
    assert (layers[0].spec.pad_h, layers[0].spec.pad_w) == (1, 1)
    assert (layers[1].spec.pad_h, layers[1].spec.pad_w) == (0, 3) and layers[1].spec.N == 2
    for bad in ("C,K\n1,2\n", "id,C\n1,2,3\n", "id,C,K,H,W,R,S,stride\n", "id,C,K,H,W,R,S,stride\n1,a,1,1,1,1,1,1\n",
                "id,C,K,H,W,R,S,stride\n1,4,4,4,4,7,7,1,0,0\n"):
        with pytest.raises(dconv.ParseError):
            lb.parse_layer_csv(bad, 1)
    assert [e.id for e in lb.builtin_resnet50(1)] == list(range(1, 21))


def test_report_json_and_csv_schema(dconv):
    from paper_1808_05567_b200 import layer_bench as lb

    s = dconv.make_layer_spec(2, 64, 64, 56, 56, 3, 3, 1)
    lr = lb.LayerReport(4, s, flops=dconv.pass_flops(s), best_ms=1.0, avg_ms=1.5, gflops=2.0, samples=3,
                        checked=True, check_ok=True,
                        norms={"linf_abs": 1e-6, "l2_abs": 1e-5, "linf_rel": 1e-7, "l2_rel": 1e-8},
                        blocking={"mb": 2}, strategy="copy_reduce", copies=8, route="duality_stride1")
    rep = lb.BenchReport("resnet50", 2, 3, "F", "f32", per_layer=[lr])
    j = lb.report_json(rep)
    assert set(j) == {"layers", "minibatch", "iterations", "pass", "impl", "dtype", "threads", "seed", "all_ok",
                      "results"}
    r = j["results"][0]
    for k in ("id", "C", "K", "H", "W", "R", "S", "stride", "pad_h", "pad_w", "flops", "best_ms", "avg_ms", "gflops",
              "samples", "check_ok", "linf_abs", "l2_abs", "linf_rel", "l2_rel", "blocking", "strategy", "copies",
              "route"):
        assert k in r, k
    assert r["flops"] == 2 * 2 * 64 * 64 * 56 * 56 * 9
    out = io.StringIO()
    lb.write_report_csv(rep, out)
    head, row = out.getvalue().splitlines()
    assert head == "id,C,K,H,W,R,S,stride,pad_h,pad_w,flops,best_ms,avg_ms,gflops,check_ok,linf_abs,l2_abs,linf_rel,l2_rel"
    assert len(row.split(",")) == 19
    buf = io.StringIO()
    lb.print_report(rep, buf)
    assert "GFLOPS" in buf.getvalue() and "ok" in buf.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("pass_", ["F", "B", "U"])
def test_layer_bench_checked_run(dconv, tmp_path, pass_):
    from paper_1808_05567_b200 import layer_bench as lb

    csv_path = tmp_path / "layers.csv"
    csv_path.write_text("id,C,K,H,W,R,S,stride\n4,64,64,56,56,3,3,1\n11,512,1024,28,28,1,1,2\n")
    out = tmp_path / "r.json"
    rc = lb.main(["--layers", str(csv_path), "--minibatch", "2", "--iters", "2", "--pass", pass_, "--check",
                  "--out", str(out), "--csv", str(tmp_path / "r.csv")] + (["--fuse", "relu"] if pass_ == "F" else []))
    assert rc == 0
    j = json.loads(out.read_text())
    assert j["all_ok"] and len(j["results"]) == 2 and all(r["gflops"] > 0 for r in j["results"])


@pytest.mark.gpu
def test_layer_bench_chain(dconv, tmp_path):
    from paper_1808_05567_b200 import layer_bench as lb

    csv_path = tmp_path / "chain.csv"
    csv_path.write_text("id,C,K,H,W,R,S,stride\n1,16,32,20,20,3,3,1\n2,32,48,20,20,1,1,2\n3,48,16,10,10,3,3,1\n")
    assert lb.main(["--layers", str(csv_path), "--minibatch", "2", "--chain", "--check"]) == 0
