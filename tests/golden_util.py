"""Helpers to load the golden vectors recorded from the unmodified reference."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def index():
    return json.loads((GOLDEN / "index.json").read_text())


def cases():
    return [k for k in index() if k != "kat"]


def load(tag):
    d = dict(np.load(GOLDEN / f"{tag}.npz"))
    d["labels"] = np.unpackbits(d.pop("labels_packed"))[: int(d.pop("n_labels"))]
    for k in ("eval_counts", "stats"):
        if k in d:
            d[k] = json.loads(str(d[k]))
    return d


def field_of(tag):
    from paper_2409_13418_b200.fields import Scene, field_from_dict

    meta = index()[tag]
    scene, R = meta["scene"], meta["R"]
    f = field_from_dict(scene["field"])
    dom = scene.get("domain", {})
    sc = Scene(f, smooth_k=scene.get("smooth_k"), domain_lo=dom.get("lo", (0, 0, 0)), domain_hi=dom.get("hi", (1, 1, 1)))
    lo, hi = tuple(sc.domain_lo.tolist()), tuple(sc.domain_hi.tolist())
    h = (np.asarray(hi) - np.asarray(lo)) / R
    return sc.resolve_field(h), lo, hi, R
