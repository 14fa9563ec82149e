"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
host-side logic mirrors the reference, and the product path fails loudly
without a GPU (no CPU fallback)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "dmlp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dmlp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_1003_0358_b200 import _lib

    lib = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    # the ctypes signature table covers exactly the header
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == syms


def test_library_is_sm100a():
    import subprocess

    from paper_1003_0358_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch

    from paper_1003_0358_b200.device import DeviceNet

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        DeviceNet((841, 10, 10))


def test_architecture_and_counts(golden):
    from paper_1003_0358_b200.network import Architecture, count_weights

    g = golden("eval")
    cfgs = [(841, 1000, 500, 10), (841, 1500, 1000, 500, 10), (841, 2000, 1500, 1000, 500, 10),
            (841, 2500, 2000, 1500, 1000, 500, 10), (841,) + (1000,) * 9 + (10,)]
    assert [count_weights(Architecture(c)) for c in cfgs] == list(g["count_weights"])
    assert Architecture.parse("841, 70,10").layer_sizes == (841, 70, 10)
    assert Architecture((841, 70, 10)).layer_shapes() == [(70, 842), (10, 71)]
    with pytest.raises(ValueError):
        Architecture((841,))
    with pytest.raises(ValueError):
        Architecture((841, 0, 10))


def test_scaled_tanh_known_answers(golden):
    from paper_1003_0358_b200.network import scaled_tanh, scaled_tanh_derivative

    g = golden("eval")
    assert scaled_tanh(1.5) == float(g["scaled_tanh_1p5"])
    assert scaled_tanh_derivative(0.0) == float(g["deriv_0"])


def test_checkpoint_roundtrip_and_errors():
    from paper_1003_0358_b200.errors import CorruptHeader, PayloadLengthMismatch, VersionMismatch
    from paper_1003_0358_b200.network import (Architecture, init_mlp, load_checkpoint,
                                              save_checkpoint)
    from paper_1003_0358_b200.rng import substream

    mlp = init_mlp(substream(0, 1), Architecture((841, 20, 10)))
    blob = save_checkpoint(mlp, 3, 1.25)
    ck = load_checkpoint(blob)
    assert ck.epoch == 3 and ck.validation_error == 1.25
    for a, b in zip(ck.mlp.layers, mlp.layers):
        assert np.array_equal(a, b)
    with pytest.raises(CorruptHeader):
        load_checkpoint(b"DM")
    with pytest.raises(CorruptHeader):
        load_checkpoint(b"XXXX" + blob[4:])
    with pytest.raises(VersionMismatch):
        load_checkpoint(blob[:4] + b"\x02\x00" + blob[6:])
    with pytest.raises(PayloadLengthMismatch):
        load_checkpoint(blob[:-4])


def test_checkpoint_matches_reference_bytes():
    """Byte-identical to the reference's save_checkpoint (network.py:156-168)."""
    import struct

    from paper_1003_0358_b200.network import Architecture, init_mlp, save_checkpoint
    from paper_1003_0358_b200.rng import substream

    mlp = init_mlp(substream(4, 1), Architecture((841, 7, 10)))
    head = b"DMLP" + struct.pack("<H", 1) + struct.pack("<I", 3) + struct.pack("<3I", 841, 7, 10)
    head += struct.pack("<I", 2) + struct.pack("<d", 0.5)
    want = head + b"".join(np.ascontiguousarray(w, dtype="<f4").tobytes() for w in mlp.layers)
    assert save_checkpoint(mlp, 2, 0.5) == want


def test_init_matches_oracle():
    from oracle import oracle as O
    from paper_1003_0358_b200.network import Architecture, init_mlp
    from paper_1003_0358_b200.rng import substream

    sizes = (841, 70, 33, 10)
    got = init_mlp(substream(0, 1), Architecture(sizes)).layers
    for a, b in zip(got, O.init_layers(0, sizes)):
        assert np.array_equal(a, b)


def test_rng_keys(golden):
    from paper_1003_0358_b200.rng import stream_key, substream

    g = golden("rng")
    pos = 0
    for k, L in enumerate(g["path_len"]):
        path = [int(v) for v in g["path_flat"][pos:pos + L]]
        pos += L
        assert stream_key(path[0], *path[1:]) == tuple(int(v) for v in g["keys"][k])
    assert np.array_equal(substream(0, 2, 0, 0).bit_generator.random_raw(16), g["words"])


def test_lr_schedule_and_config(golden):
    from paper_1003_0358_b200.network import Architecture
    from paper_1003_0358_b200.trainer import TrainConfig, lr_schedule

    g = golden("eval")
    cfg = TrainConfig(arch=Architecture((841, 70, 33, 10)))
    got = [lr_schedule(e, cfg) for e in (0, 1, 10, 100, 982, 983, 2000)]
    assert np.array_equal(np.array(got), g["lr"])
    for bad in [dict(eta0=0.0), dict(decay=1.0), dict(max_epochs=-1), dict(lanes=0),
                dict(variant="fast")]:
        with pytest.raises(ValueError):
            TrainConfig(arch=Architecture((841, 10)), **bad)
    TrainConfig(arch=Architecture((841, 10)), variant="tiled")  # reference alias accepted


def test_deform_params_validation():
    from paper_1003_0358_b200.deform import DeformParams
    from paper_1003_0358_b200.errors import EvenSize, InvalidSigma

    with pytest.raises(InvalidSigma):
        DeformParams(sigma_range=(0.0, 1.0))
    with pytest.raises(EvenSize):
        DeformParams(kernel_size=20)
    with pytest.raises(ValueError):
        DeformParams(alpha_range=(2.0, 1.0))
    ident = DeformParams.identity()
    assert ident.alpha_range == (0.0, 0.0) and ident.beta_default == 0.0


def test_rank_outputs_ties():
    from paper_1003_0358_b200.network import rank_outputs

    y = np.array([[0.1, 0.5, 0.5, -1.0], [0.3, 0.3, 0.3, 0.3]], dtype=np.float32)
    r = rank_outputs(y)
    assert list(r[0][:3]) == [1, 2, 0]
    assert list(r[1]) == [0, 1, 2, 3]


def test_synthetic_digits_deterministic():
    from paper_1003_0358_b200.synthetic import make_digits

    a, la = make_digits(300, seed=5)
    b, lb = make_digits(300, seed=5)
    assert np.array_equal(a, b) and np.array_equal(la, lb)
    assert a.dtype == np.uint8 and a.shape == (300, 28, 28)
    assert set(np.unique(la)) <= set(range(10))
    assert 10 < a.mean() < 80


def test_idx_roundtrip():
    from paper_1003_0358_b200.mnist_io import BadMagic, parse_idx_images, parse_idx_labels
    from paper_1003_0358_b200.synthetic import make_digits, write_idx_images, write_idx_labels

    im, lab = make_digits(20, seed=1)
    assert np.array_equal(parse_idx_images(write_idx_images(im)), im)
    assert np.array_equal(parse_idx_labels(write_idx_labels(lab)), lab)
    with pytest.raises(BadMagic):
        parse_idx_images(write_idx_labels(lab))


def test_shard_range_partitions():
    from paper_1003_0358_b200.distributed import shard_range

    for n in (0, 1, 7, 60000, 10001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_bench_gpus_flag_relaunches_under_torchrun():
    """`bench.py --gpus 2` started without torchrun re-launches itself as two
    ranks (the driver's own launch); the reference arm then prints one line
    from rank 0 only, with n_gpus = 2 (runs on CPU: the reference arm is the
    oracle port)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "3", "--cpu-seconds", "0.5"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"


def test_bench_level_bytes_split():
    """bench.py's hybrid roofline: 12 B per weight by the level that serves it --
    register columns and the register plan's smem tail, smem layers, and a
    streamed layer split between L1 (its L1-served rows per CTA) and L2; the
    output tile counts as smem.  Every weight is counted once."""
    import importlib.util
    import types

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    sizes = (841, 2500, 2000, 1500, 1000, 500, 10)
    dn = types.SimpleNamespace(
        layer_residency=["smem", "reg", "smem", "l2", "smem", "smem"],
        layer_reg_cols=[0, 2048, 0, 0, 0, 0], layer_l1_rows=[0, 0, 0, 5, 0, 0], n_ctas=148)
    lv = bench.level_bytes(sizes, dn)
    W = sum((i + 1) * o for i, o in zip(sizes[:-1], sizes[1:]))
    assert sum(lv.values()) == 12 * W
    assert lv["reg"] == 12 * 2000 * 2048
    l3 = 12 * 1000 * 1501
    assert lv["l1"] == int(l3 * 5 / 7) and lv["l2"] == l3 - lv["l1"]
