"""compute-sanitizer checks of the persistent training kernel (B200).

The flag-word exchanges leave the lanes of a warp in different poll rounds;
the CTA barriers after them must tolerate that (train_phases.cuh cta_sync).
synccheck catches a barrier reached by a divergent warp -- the failure that
made the register-only instance compute wrong weights -- and racecheck the
shared-memory hazards between the phases.  Each check runs a few samples of
a small net in a subprocess, once per compiled feature instance (register
rows only; smem + L2 paths forced in with DMLP_RES_ALLPATHS).
"""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from oracle import oracle as O
from paper_1003_0358_b200.device import DeviceNet
g = np.load(%r); x = g['deformed'].reshape(64, -1); lab = g['labels']
sizes = tuple(int(v) for v in sys.argv[1].split(','))
n = int(sys.argv[2])
dn = DeviceNet(sizes, all_paths=sys.argv[3] == '3'); dn.set_layers(O.init_layers(7, sizes))
wrong = torch.zeros((), dtype=torch.int64, device='cuda')
dn.train_epoch(torch.from_numpy(x[:n]).cuda(), torch.from_numpy(lab[:n]).cuda(), None, 1e-3, wrong)
torch.cuda.synchronize()
print('ok', ''.join(r[0] for r in dn.layer_residency))
""" % (ROOT, os.path.join(ROOT, "tests", "golden", "train.npz"))


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    pytest.skip("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["synccheck", "racecheck"])
@pytest.mark.parametrize("feat", ["0", "3"])
@pytest.mark.parametrize("sizes", ["841,300,120,10", "841,37,5,9,10"])
def test_train_kernel_sanitizer(tmp_path, tool, feat, sizes):
    script = tmp_path / "case.py"
    script.write_text(CASE)
    p = subprocess.run([_sanitizer(), "--tool", tool, "--print-limit", "4", "--error-exitcode", "9",
                        sys.executable, str(script), sizes, "3", feat],
                       capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "ok " in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards" in out, out[-3000:]


@pytest.mark.parametrize("tool", ["synccheck", "racecheck", "memcheck"])
def test_train_kernel_l1_instance_sanitizer(tmp_path, tool):
    """The headline net's auto plan runs the L1-feature instance (layer 3's
    first rows per thread through L1): two samples under each tool."""
    script = tmp_path / "case.py"
    script.write_text(CASE)
    p = subprocess.run([_sanitizer(), "--tool", tool, "--print-limit", "4", "--error-exitcode", "9",
                        sys.executable, str(script), "841,2500,2000,1500,1000,500,10", "2", "0"],
                       capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "ok " in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards" in out, out[-3000:]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_deform_eval_sanitizer(tool):
    """memcheck / racecheck of the deformation (4 images per CTA, ragged last
    batch, unaligned raw rows, another kernel size), upscale and evaluation
    (padded-input GEMM path) kernels: scripts/memcheck_deform_eval.py."""
    p = subprocess.run([_sanitizer(), "--tool", tool, "--print-limit", "4", "--error-exitcode", "9",
                        sys.executable, os.path.join(ROOT, "scripts", "memcheck_deform_eval.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "ok " in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards" in out, out[-3000:]
