"""GPU: K4 splits batches whose TMA row coordinates would pass 2^31 into
several launches (tfft_k3.cu k4_execute). The split is forced small through
TFFT_K4_MAX_BATCH in a subprocess: outputs must be bitwise equal to one
launch, and a stage-0 fault in a later chunk must still strike its signal."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2412_05824_b200 as tf
from conftest import gaussian
for prec, n, b in (("double", 16384, 37), ("single", 65536, 23)):
    x = gaussian(n, b, prec, seed=5)
    plan = tf.build_plan(tf.select_params(n, b, prec), prec)
    y = tf.execute_plan(plan, tf.SignalBatch(x)).data
    spec = tf.FaultSpec(transaction=(b - 3) // plan.bs, signal=b - 3, element=n // 5, stage=0, part="im", bit=20)
    inj = tf.FaultInjector(); inj.arm(spec, plan=plan, batch=tf.SignalBatch(x))
    yf = tf.execute_plan(plan, tf.SignalBatch(x), injector=inj).data
    np.save(sys.argv[1] + "_%%s_y.npy" %% prec, y)
    np.save(sys.argv[1] + "_%%s_yf.npy" %% prec, yf)
"""


def _run(tmp, env_extra):
    env = dict(os.environ, **env_extra)
    code = SCRIPT % (str(ROOT), str(ROOT / "tests"))
    subprocess.run([sys.executable, "-c", code, str(tmp)], check=True, env=env, cwd=ROOT)


def test_k4_chunked_launches_bitwise(tmp_path):
    import numpy as np
    _run(tmp_path / "one", {})
    _run(tmp_path / "chunks", {"TFFT_K4_MAX_BATCH": "5"})
    for prec in ("double", "single"):
        y1 = np.load(str(tmp_path / "one") + f"_{prec}_y.npy")
        y2 = np.load(str(tmp_path / "chunks") + f"_{prec}_y.npy")
        assert np.array_equal(y1, y2)
        f1 = np.load(str(tmp_path / "one") + f"_{prec}_yf.npy")
        f2 = np.load(str(tmp_path / "chunks") + f"_{prec}_yf.npy")
        assert np.array_equal(f1, f2)
        changed = np.nonzero(np.any(f1 != y1, axis=1))[0]
        assert list(changed) == [y1.shape[0] - 3]
