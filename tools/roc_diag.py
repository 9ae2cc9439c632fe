"""Diagnostic (GPU): run the 2000-trial ROC protocol and print where our
per-trial divergences depart from the reference fixture's."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_2412_05824_b200 as tf
    ref = json.loads((ROOT / "tests/golden/golden_scale.json").read_text())["roc"]
    cfg = tf.CampaignConfig(**{**ref["config"], "delta_sweep": tuple(ref["config"]["delta_sweep"])})
    res = tf.roc_campaign(cfg)
    print("ours rows", res.rows)
    print("ref  rows", ref["rows"])
    ours = np.array([t.divergence for t in res.trials])
    theirs = np.array([r[2] for r in ref["trials"]])
    inj = np.array([r[0] for r in ref["trials"]])
    for name, m in (("clean", ~inj), ("injected", inj)):
        print(name, "ours pct", np.percentile(ours[m], [0, 1, 50, 99, 100]), "ref pct",
              np.percentile(theirs[m], [0, 1, 50, 99, 100]))
    ratio = ours / np.maximum(theirs, 1e-30)
    print("ratio ours/ref clean pct", np.percentile(ratio[~inj], [1, 50, 99]))
    for t in res.trials:
        r = ref["trials"][t.trial]
        if t.injected and (not np.isfinite(t.divergence) or t.divergence < 2e-7 or abs(t.divergence / max(r[2], 1e-30) - 1) > 0.5):
            print("trial", t.trial, "bit", t.bit, "ours", t.divergence, "ref", r[2], "det", t.detected, r[3])


if __name__ == "__main__":
    main()
