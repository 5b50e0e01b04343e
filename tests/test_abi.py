"""CPU-side checks of the C ABI: the library loads, exports every symbol the header
declares, and its host functions (tap tables, angle assignment, validation) agree
with the oracle.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import taps as T
from paper_2309_15812_b200 import binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2309_15812_b200 import build
    build.build()
    B.lib()


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "oriented1d.h")).read()
    declared = set(re.findall(r"O1D_API[^;(]*?\b(o1d_\w+)\s*\(", hdr))
    assert len(declared) >= 16
    L = ctypes.CDLL(B.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert set(B.EXPORTS) == declared
    assert "sm_100a" in B.version()


def _angle_sets():
    sets = {}
    for D in (2, 4, 8):
        for assign in ("contiguous", "cycled"):
            sets[f"D{D}_{assign}"] = T.direction_angles(D, 8 * D, assign)
    for C in (8, 96, 128, 192, 256, 384, 512, 768, 1024):
        sets[f"D=C={C}"] = T.direction_angles(C, C)
    sets["integer_deg"] = [float(a) for a in range(360)]
    sets["half_deg"] = [a * 0.5 for a in range(720)]
    sets["negative"] = [-a * 7.5 for a in range(48)]
    eps = [1e-3, 1e-6, 1e-9, 1e-12]
    sets["near_niven"] = [a + s * e for a in (0, 30, 60, 90, 120, 150, 180, 210, 270, 330)
                          for e in eps for s in (-1, 1)]
    sets["big"] = [725.5, -3600.0, 1e3, 1e6 + 0.5, -1e5 - 30.0]
    return sets


@pytest.mark.parametrize("K", [3, 5, 7, 15, 27, 31, 63])
def test_make_taps_bit_exact_vs_oracle(K):
    """T1: the library's f64+snap tap generator equals the exact-math oracle bit for bit."""
    for name, angles in _angle_sets().items():
        oh, ow = B.make_taps(K, np.array(angles))
        roh, row = T.taps_table(K, K // 2, angles)
        assert np.array_equal(oh, np.array(roh, np.int16)), (name, K)
        assert np.array_equal(ow, np.array(row, np.int16)), (name, K)


def test_make_taps_nondefault_pad():
    angles = np.array([0.0, 22.5, 30.0, 45.0, 60.0, 90.0, 135.0, 150.0, 300.0, 17.3])
    for K, pad in ((7, 0), (7, 6), (8, 4), (6, 2), (6, 2.5), (7, 1.25), (31, 14.5), (4, 0.5)):
        oh, ow = B.make_taps(K, angles, pad=pad)
        roh, row = T.taps_table(K, pad, angles)
        assert np.array_equal(oh, np.array(roh)) and np.array_equal(ow, np.array(row)), (K, pad)


@pytest.mark.parametrize("K", [3, 7, 15, 31])
def test_make_bilinear_vs_oracle(K):
    """Bilinear tables: base corners bit-exact, fractional parts within 1e-14 of
    the oracle's 80-digit values (exactly 0 / 1/2 at the Niven angles)."""
    sets = _angle_sets()
    for name in ("D8_cycled", "D=C=96", "integer_deg", "near_niven", "big"):
        angles = sets[name]
        h0, w0, fa, fb = B.make_bilinear(K, np.array(angles))
        rh, rw, ra, rb = (np.array(v) for v in T.bilinear_table(K, K // 2, angles))
        assert np.array_equal(h0, rh) and np.array_equal(w0, rw), name
        assert np.max(np.abs(fa - ra)) < 1e-14 and np.max(np.abs(fb - rb)) < 1e-14, name
        exact = np.isin(np.array(angles) % 360.0, [0.0, 30.0, 90.0, 150.0, 180.0, 210.0, 270.0, 330.0])
        assert np.array_equal(fa[exact], ra[exact]), name


def test_direction_angles_vs_oracle():
    for D, C in ((4, 8), (8, 96), (8, 384), (96, 96), (768, 768), (2, 4)):
        for assign in ("contiguous", "cycled"):
            for shift in (0.0, 90.0):
                got = B.direction_angles(D, C, assign, shift)
                assert got.tolist() == T.direction_angles(D, C, assign, shift), (D, C, assign, shift)


def test_error_codes():
    with pytest.raises(B.O1DError) as e:
        B.direction_angles(3, 8)
    assert e.value.status == 3 and "divide" in str(e.value)
    with pytest.raises(B.O1DError) as e:
        B.make_taps(0, np.zeros(2))
    assert e.value.status == 3
    L = B.lib()
    h = ctypes.c_void_p()
    ang = np.zeros(4)
    for fields, status in (((0, 4, 8, 8, 3, 1, -1, 0, 0, 0), 2),  # N = 0
                           ((1, 4, 8, 8, 0, 1, -1, 0, 0, 0), 3),  # K = 0
                           ((1, 4, 8, 8, 3, 0, -1, 0, 0, 0), 3),  # stride 0
                           ((1, 4, 8, 8, 3, 1, 3, 0, 0, 0), 3),   # pad > K - 1
                           ((1, 4, 8, 8, 3, 1, 2.5, 0, 0, 0), 3),  # pad > K - 1 (real)
                           ((1, 4, 8, 8, 3, 1, float("nan"), 0, 0, 0), 1),  # non-finite pad
                           ((1, 4, 8, 8, 3, 1, 1.5, 0, 0, 4), 5),  # shear with a non-integer pad
                           ((1, 4, 8, 8, 3, 1, -1, 0, 0, 12), 3),  # shear and bilinear
                           ((1, 4, 8, 8, 3, 1, -1, 7, 0, 0), 5),  # dtype
                           ((1, 4, 8, 8, 3, 1, -1, 0, 1, 0), 5)):  # layout
        d = B._Desc(*fields)
        st = L.o1d_plan_create(ctypes.byref(d), B._ptr(ang), ctypes.byref(h))
        assert st == status, (fields, st, L.o1d_last_error())
        assert not h.value
    assert L.o1d_forward(None, None, None, None, None) == 1


@pytest.mark.parametrize("disc", ["rotation", "bilinear"])
@pytest.mark.parametrize("pass_id", [0, 1, 2, 3])
def test_spec_source_compiles_for_sm100a(tmp_path, pass_id, disc):
    """The runtime-generated specialised kernels are valid sm_100a CUDA (host-only
    generation through the ABI, compiled here with nvcc; no GPU needed); pass 3 is the
    fused backward (NEXT-2)."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    flags = B.FLAG_BILINEAR if disc == "bilinear" else 0
    src = B.spec_source(2, 16, 56, 56, 15, T.direction_angles(8, 16, "cycled"), pass_id, flags=flags)
    assert "o1d_" in src and "cp.async.bulk.tensor" in src
    f = tmp_path / f"k{pass_id}.cu"
    f.write_text(src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-o", str(tmp_path / "k.cubin"),
                        str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    sass = subprocess.run(["cuobjdump", "-sass", str(tmp_path / "k.cubin")], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass and "FFMA2" in sass  # TMA tile loads, packed FP32
    if pass_id != 2:
        assert "UTMASTG" in sass  # TMA band stores


def test_spec_source_ineligible_shapes():
    with pytest.raises(B.O1DError) as e:
        B.spec_source(1, 8, 30, 30, 7, np.zeros(8), 0)  # 30*4 B rows: not TMA-legal, too big for small planes
    assert e.value.status == 5
    with pytest.raises(B.O1DError):
        B.spec_source(1, 8, 15, 15, 7, np.zeros(8), 0)  # 15 > 14 and 60-byte rows: generic kernels
    with pytest.raises(B.O1DError):
        B.spec_source(1, 8, 56, 56, 7, np.zeros(8), 0, stride=2)


def test_make_taps_shear_bit_exact():
    """The library's shear-form tables (o1d_make_taps_ex) equal the oracle's exact
    tables bit for bit, incl. angles within 1e-7 deg of the 45-degree family (tan = +-1)."""
    import random
    from oracle import taps as T
    rnd = random.Random(3)
    angs = [0, 45, 90, 135, 180, -45, 22.5, 67.5, 112.5, 157.5, 30, 60, 89.999, 90.001, 44.9999999,
            45.0000001, 134.9999999, 1e-9, -1e-9, 359.99999] + [rnd.uniform(-720, 720) for _ in range(200)]
    angs += [i * 180 / 96 for i in range(96)] + list(range(0, 360, 7))
    for K in (1, 3, 7, 31, 63):
        oh, ow = B.make_taps(K, np.array(angs, float), discretization="shear")
        roh, row = T.taps_table(K, K // 2, angs, "shear")
        assert np.array_equal(oh, np.array(roh)) and np.array_equal(ow, np.array(row)), K
    with pytest.raises(ValueError):
        B.make_taps(7, np.zeros(2), discretization="nonsense")
    import ctypes
    a = np.zeros(2)
    o1, o2 = np.empty((2, 7), np.int16), np.empty((2, 7), np.int16)
    assert B.lib().o1d_make_taps_ex(7, 3, 2, a.ctypes.data, 5, o1.ctypes.data, o2.ctypes.data) == 1  # INVALID_ARG


@pytest.mark.parametrize("dtype,pass_id", [("f32", 0), ("f32", 2), ("bf16", 1)])
def test_small_plane_source_compiles_for_sm100a(tmp_path, pass_id, dtype):
    """Planes of at most 14 x 14 get the small-plane kernels (32-plane items, compile-time block
    positions, exact pruning of out-of-image taps): valid sm_100a code, TMA box loads for fp32
    planes of 16-byte multiples, cp.async (LDGSTS) units otherwise, packed FP32 in the tap code."""
    import shutil
    import subprocess
    import torch
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    dt = torch.float32 if dtype == "f32" else torch.bfloat16
    src = B.spec_source(128, 16, 14, 14, 31, T.direction_angles(4, 16, "cycled"), pass_id, dtype=dt)
    assert "o1d_small" in src
    f = tmp_path / f"s{pass_id}.cu"
    f.write_text(src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-o", str(tmp_path / "s.cubin"),
                        str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    sass = subprocess.run(["cuobjdump", "-sass", str(tmp_path / "s.cubin")], capture_output=True, text=True).stdout
    assert "FFMA2" in sass
    assert ("UTMALDG" in sass) == (dtype == "f32") and ("LDGSTS.E" in sass) == (dtype != "f32" or pass_id <= 1)


@pytest.mark.parametrize("pass_id", [0, 2])
def test_flat_16bit_source_compiles_for_sm100a(tmp_path, pass_id):
    """16-bit planes whose rows are not 16-byte multiples (ConvNeXt stage 2: 28 x 2 B) get the
    specialised kernels through flat TMA views (planes as rows of 8 elements); 30-wide planes (rows of
    4-element units do not fit) stay on the generic kernels."""
    import shutil
    import subprocess
    import torch
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    src = B.spec_source(4, 16, 28, 28, 31, T.direction_angles(8, 16, "cycled"), pass_id, dtype=torch.bfloat16)
    if pass_id == 0:
        assert "row0 * 14 / 4" in src  # band store at element row0 * 28 / 8 of the flat view
    f = tmp_path / f"f{pass_id}.cu"
    f.write_text(src)
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-o", str(tmp_path / "f.cubin"),
                        str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    with pytest.raises(B.O1DError):
        B.spec_source(4, 16, 30, 30, 31, T.direction_angles(8, 16, "cycled"), pass_id, dtype=torch.bfloat16)


def test_wgrad_pair_step_selection(monkeypatch):
    """backward_weight packs tap pairs along the step with the fewest generated FMA instructions
    (16 candidates): the same FMA count as the round-1 candidate set (4 steps), never more
    instructions, strictly fewer for the near-22.5 deg tables of D=8."""
    import re

    def counts(n):
        monkeypatch.setenv("O1D_PPSTEPS", str(n))
        src = B.spec_source(2, 16, 56, 56, 31, T.direction_angles(8, 16, "cycled"), 2)
        out = []
        for body in re.split(r"\n    case \d+: \{", src)[1:]:
            body = body.split("break;")[0]
            f2, f1 = body.count("ffma2("), body.count("fmaf(")
            out.append((2 * f2 + f1, f2 + f1))
        return out

    c16, c4 = counts(16), counts(4)
    assert len(c16) == len(c4) == 8
    for (fma16, ins16), (fma4, ins4) in zip(c16, c4):
        assert fma16 == fma4 and ins16 <= ins4
    assert sum(i for _, i in c16) < sum(i for _, i in c4)
