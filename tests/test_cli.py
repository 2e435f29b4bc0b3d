"""Command-line driver (occmesh.cli, cli.py:1-305) on the GPU path: same
options, report document and exit codes as the reference's driver (golden
reports in tests/golden/cli_golden.json, made by make_cli_golden.py)."""

import json
from pathlib import Path

import pytest

from paper_2409_13418_b200 import scenes
from paper_2409_13418_b200.cli import RunConfig, build_parser, parse_method

GOLDEN = Path(__file__).resolve().parent / "golden"
RUNS = json.loads((GOLDEN / "cli_golden.json").read_text())


@pytest.mark.parametrize("method,kind,detail", [
    ("odc", "stage", ("binary-search", "two-d-points", "ic")),
    ("ic", "stage", ("binary-search", "two-d-points", "ic")),
    ("mc", "mc", "binary"),
    ("mc:continuous", "mc", "continuous"),
    ("stage:linear,fd,mdc", "stage", ("linear-interp", "fd-gradient", "mdc")),
    ("stage:midpoint,2d,ic", "stage", ("midpoint", "two-d-points", "ic")),
])
def test_parse_method(method, kind, detail):
    k, stage, mode = parse_method(RunConfig(scene="x", method=method))
    assert k == kind
    assert (mode if kind == "mc" else (stage.one_d, stage.normals, stage.split)) == detail


@pytest.mark.parametrize("method", ["bogus", "stage:a,b", "stage:linear,fd,xyz"])
def test_parse_method_errors(method):
    from paper_2409_13418_b200 import ConfigurationError

    with pytest.raises(ConfigurationError):
        parse_method(RunConfig(scene="x", method=method))


def test_parser_has_reference_options():
    a = build_parser().parse_args(["run", "--scene", "s.json"])
    for k in ("resolution", "method", "out", "report", "gt", "iters_1d", "step1_linear", "step1_binary", "step1_range",
              "step2_linear", "step2_binary", "step2_range", "qef_truncation", "no_ic", "mc_mode", "metric_samples",
              "seed", "threads", "allow_nonmanifold", "max_si"):
        assert hasattr(a, k), k


EXACT = ("n_vertices", "n_triangles", "manifold", "si_count", "euler_characteristic", "eval_counts", "open_boundary",
         "warnings", "split_case_counts", "qef_rank_counts", "normal_fallbacks", "schema_version", "method_resolved",
         "config")


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(RUNS))
def test_gpu_cli_matches_reference(tmp_path, key):
    from paper_2409_13418_b200.cli import main

    scene, R, method, _ = key.split("|")
    run = RUNS[key]
    sp = tmp_path / "scene.json"
    sp.write_text(json.dumps(scenes.SCENES[scene]))
    extra = [str(GOLDEN / "cli_gt_sphere40.obj") if x == "GT" else x for x in run["extra"]]
    rp = tmp_path / "report.json"
    code = main(["run", "--scene", str(sp), "--resolution", R, "--method", method, "--report", str(rp),
                 "--metric-samples", "4000", "--allow-nonmanifold", "--max-si", "1000", "--out",
                 str(tmp_path / "m.obj")] + extra)
    assert code == run["exit"]
    if run["report"] is None:
        assert not rp.exists()
        return
    doc = json.loads(rp.read_text())
    for k in ("scene", "out", "report", "gt"):
        doc["config"].pop(k)
    want = run["report"]
    # the reference serialises eval-count and histogram keys via json (ints -> strings)
    doc = json.loads(json.dumps(doc))
    for k in EXACT:
        assert doc[k] == want[k], k
    for k in ("qef_max_residual", "fit_err", "md2", "nic", "hdd"):
        a, b = doc.get(k), want.get(k)
        assert (a is None) == (b is None), k
        if a is not None:
            assert abs(a - b) <= 1e-6 * max(abs(b), 1e-12), (k, a, b)
    assert (tmp_path / "m.obj").exists()
