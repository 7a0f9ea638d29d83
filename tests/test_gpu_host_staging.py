"""GPU: host (pinned and pageable) buffers through the C ABI with many staging chunks --
INFT_STAGE_MB=1 forces chunks of a few RHS, so the double-buffered H2D / compute / D2H
pipeline, the quarter-size first and last chunks (INFT_STAGE_RAMP) and the uniform schedule
all run; results equal the device-buffer path to rounding (a chunk's row-group count sets the
ring chunk tables, hence the summation order of split segments) and the oracle within the
parity bar.  Run in a subprocess: the knobs are read once."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch
import oracle as O, synth as S, paper_1811_05335_b200 as P
M, sigma, m, N, R = 4096, 2.0, 8, 8192, 45     # f row 128 KB: 1 MB chunks = 8 RHS
x = S.jittered(N, 3)
live = O.slot_live(x, O.msigma(M, sigma), m)
w = np.random.default_rng(1).standard_normal(live.shape) * live
plan = P.Plan(x, M, sigma, m).set_bopt(w, "alg2")
f = S.normal_complex(R, N, 5)
h = S.normal_complex(R, M, 6)
dev_i = plan.apply(torch.from_numpy(f).cuda()).cpu().numpy()
dev_a = plan.adjoint_apply(torch.from_numpy(h).cuda()).cpu().numpy()
for pinned in (False, True):
    fi = torch.from_numpy(f).pin_memory() if pinned else f
    hi = torch.from_numpy(h).pin_memory() if pinned else h
    oi = plan.apply(fi)
    oa = plan.adjoint_apply(hi)
    oi = oi.numpy() if hasattr(oi, "numpy") else oi
    oa = oa.numpy() if hasattr(oa, "numpy") else oa
    assert O.rel_l2(oi, dev_i) <= 1e-14 and O.rel_l2(oa, dev_a) <= 1e-14, pinned
ref_i = O.apply_inverse(x, M, sigma, m, w, 1.0, f)
ref_a = O.apply_adjoint(x, M, sigma, m, w, 1.0, h)
assert O.rel_l2(dev_i, ref_i) <= 1e-12 and O.rel_l2(dev_a, ref_a) <= 1e-12
print("ok")
"""


@pytest.mark.parametrize("ramp", ["1", "0"])
def test_host_staging_chunks(ramp):
    env = dict(os.environ, INFT_STAGE_MB="1", INFT_STAGE_RAMP=ramp,
               PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]
