"""Golden reports of the reference's command-line driver (occmesh.cli.run,
cli.py:117-218) for a few scenes and methods, run here; wall time and paths
are dropped.

    python tests/golden/make_cli_golden.py
"""
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))
from occmesh.cli import main  # noqa: E402

from paper_2409_13418_b200 import scenes as SC  # noqa: E402

RUNS = [("sphere", 32, "odc", []), ("torus", 24, "mc", []), ("smooth_sphere", 24, "mc:continuous", []),
        ("rotated_box", 24, "stage:linear,fd,mdc", []), ("smooth_sphere", 24, "stage:linear,fd,mdc", []),
        ("csg_union", 24, "odc", ["--no-ic"]), ("sphere", 24, "odc", ["--gt", "GT"]),
        ("torus", 24, "bogus", [])]


def main_():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        # ground truth for the --gt run: the reference's own sphere mesh at 40^3
        (td / "sphere.json").write_text(json.dumps(SC.SCENES["sphere"]))
        main(["run", "--scene", str(td / "sphere.json"), "--resolution", "40", "--out", str(td / "gt.obj")])
        (HERE / "cli_gt_sphere40.obj").write_bytes((td / "gt.obj").read_bytes())
        for i, (scene, R, method, extra) in enumerate(RUNS):
            sp = td / f"{scene}.json"
            sp.write_text(json.dumps(SC.SCENES[scene]))
            extra = [str(td / "gt.obj") if x == "GT" else x for x in extra]
            rp = td / f"r{i}.json"
            code = main(["run", "--scene", str(sp), "--resolution", str(R), "--method", method,
                         "--report", str(rp), "--metric-samples", "4000", "--allow-nonmanifold", "--max-si", "1000"]
                        + extra)
            doc = None
            if rp.exists():
                doc = json.loads(rp.read_text())
                doc.pop("wall_time_s")
                for k in ("scene", "out", "report", "gt"):
                    doc["config"].pop(k)
            out[f"{scene}|{R}|{method}|{' '.join(x for x in extra if x != str(td / 'gt.obj'))}"] = {
                "exit": code, "extra": [("GT" if x == str(td / "gt.obj") else x) for x in extra], "report": doc}
    (HERE / "cli_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(list(out))


if __name__ == "__main__":
    main_()
