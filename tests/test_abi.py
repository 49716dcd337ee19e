"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/finom_b200.h declares; host-only entry points behave."""

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "finom_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(finom_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("finom_plan1d_create", "finom_solve1d", "finom_cost1d", "finom_apply1d",
                 "finom_iterate1d", "finom_sinkhorn1d_host", "finom_sinkhorn2d_host",
                 "finom_apply2d_host", "finom_cost2d_host"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2605_26659_b200 import _lib
    lib = _lib.load(require_device=False)
    t512 = ctypes.CDLL(_lib.LIB_T512_PATH)  # (the 512-element-tile build, _lib.lib_for)
    for name in declared():
        if name == "finom_phase_read":  # (debug builds only)
            continue
        assert hasattr(lib, name), name
        assert hasattr(t512, name), name
    assert set(_lib.SIGNATURES) >= set(declared()) - {"finom_phase_read"}
    t512.finom_build_info.restype = ctypes.c_char_p
    assert b"TILE=512" in t512.finom_build_info()
    assert "TILE=256" in lib.finom_build_info().decode()


def test_library_selection_rule(monkeypatch):
    from paper_2605_26659_b200 import _lib
    monkeypatch.delenv("FINOM_TILE", raising=False)
    assert _lib.use_t512(1, 2 * (1 << 22))        # config 2
    assert not _lib.use_t512(1, 20_000)           # config 1
    assert not _lib.use_t512(8192, 8192 * 32768)  # config 5 (the group solve)
    monkeypatch.setenv("FINOM_TILE", "512")
    assert _lib.use_t512(1, 20_000)
    monkeypatch.setenv("FINOM_TILE", "256")
    assert not _lib.use_t512(1, 2 * (1 << 22))


def test_library_is_sm100a():
    from paper_2605_26659_b200 import _lib
    info = _lib.load(require_device=False).finom_build_info().decode()
    assert "sm_100a" in info
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode == 0:
        assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device():
    """The product path fails loudly when no CUDA device is present."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2605_26659_b200 as fb
    x = fb.Mesh1D(np.linspace(0, 1, 5))
    u = fb.Measure(np.full(5, 0.2))
    with pytest.raises(fb.DeviceError):
        fb.sinkhorn_1d(x, x, u, u, fb.SolverConfig(epsilon=0.1, itr_max=3))


def _merge_ref(x, y, half):
    """Merged order bits by a plain two-pointer merge (col first on ties)."""
    bits, i, j = [], 0, 0
    while i < x.size or j < y.size:
        if half == 0:  # rows y, cols x: x_i <= y_j first
            col = i < x.size and (j == y.size or x[i] <= y[j])
            bits.append(col)
            i, j = (i + 1, j) if col else (i, j + 1)
        else:          # rows x, cols y: y_j <= x_i first
            col = j < y.size and (i == x.size or y[j] <= x[i])
            bits.append(col)
            i, j = (i, j + 1) if col else (i + 1, j)
    return bits


@pytest.mark.parametrize("n,m,ties", [(1, 1, False), (5, 3, False), (700, 900, False),
                                      (1000, 1000, True), (3000, 17, False)])
def test_tile_partition_properties(n, m, ties):
    from paper_2605_26659_b200 import _lib
    rng = np.random.default_rng(n + m)
    x = np.sort(rng.uniform(0, 1, n))
    y = x.copy() if ties else np.sort(rng.uniform(0, 1, m))
    tiles, masks = _lib.tile_partition(x, y)
    assert tiles[0, 0] == 0 and tiles[0, 2] == 0
    assert tiles[-1, 1] == x.size and tiles[-1, 3] == y.size
    for t in range(len(tiles)):
        x0, x1, y0, y1 = tiles[t]
        if t:
            assert x0 == tiles[t - 1, 1] and y0 == tiles[t - 1, 3]
        assert 0 < (x1 - x0) + (y1 - y0) <= 256
        # no tie pair split across tiles: tile elements strictly above the previous tile's
        here = np.concatenate([x[x0:x1], y[y0:y1]])
        assert here.min() > max(x[:x0].max() if x0 else -np.inf, y[:y0].max() if y0 else -np.inf)
        for half in (0, 1):
            bits = _merge_ref(x[x0:x1], y[y0:y1], half)
            word = masks[t, half * 8:(half + 1) * 8]
            got = [(int(word[k // 32]) >> (k % 32)) & 1 for k in range(len(bits))]
            assert got == [int(b) for b in bits]


@pytest.mark.parametrize("ties", [False, True])
def test_tile_partition_parallel_segments(ties):
    """Problems of >= 2^20 merged elements are tiled in 16 host-threaded segments:
    the partition stays contiguous, within the tile size, never splits a tie,
    and its merged-order masks are right at the segment joins."""
    from paper_2605_26659_b200 import _lib
    rng = np.random.default_rng(7)
    n = 600_000
    x = np.sort(rng.uniform(0, 1, n))
    y = x.copy() if ties else np.sort(rng.uniform(0, 1, n + 123))
    tiles, masks = _lib.tile_partition(x, y)
    x0, x1, y0, y1 = (tiles[:, k].astype(np.int64) for k in range(4))
    assert x0[0] == 0 and y0[0] == 0 and x1[-1] == x.size and y1[-1] == y.size
    assert np.all(x0[1:] == x1[:-1]) and np.all(y0[1:] == y1[:-1])
    sz = (x1 - x0) + (y1 - y0)
    assert sz.min() > 0 and sz.max() <= 256
    # no tie split: every element of tile t lies strictly above the last x / y before it
    lo = np.minimum(np.where(x1 > x0, x[np.minimum(x0, x.size - 1)], np.inf),
                    np.where(y1 > y0, y[np.minimum(y0, y.size - 1)], np.inf))
    prev = np.maximum(np.where(x0 > 0, x[np.maximum(x0 - 1, 0)], -np.inf),
                      np.where(y0 > 0, y[np.maximum(y0 - 1, 0)], -np.inf))
    assert np.all(lo > prev)
    # masks of the tiles around the segment joins (and a few others)
    N = x.size + y.size
    picks = {0, len(tiles) - 1}
    for s in range(1, 16):
        t = int(np.searchsorted(x0 + y0, N * s // 16, side="right")) - 1
        picks.update({max(t - 1, 0), t, min(t + 1, len(tiles) - 1)})
    for t in sorted(picks):
        for half in (0, 1):
            bits = _merge_ref(x[x0[t]:x1[t]], y[y0[t]:y1[t]], half)
            word = masks[t, half * 8:(half + 1) * 8]
            got = [(int(word[k // 32]) >> (k % 32)) & 1 for k in range(len(bits))]
            assert got == [int(b) for b in bits]


def test_fexp_host_arithmetic():
    """csrc/fexp.cuh's q_div is the IEEE quotient and fexp is within 1 ulp of libm exp."""
    exe = "/tmp/finom_fexp_check"
    src = os.path.join(ROOT, "tests", "fexp_check.cu")
    r = subprocess.run(["nvcc", "-std=c++17", "-O2", "-w", "-o", exe, src], capture_output=True,
                       text=True)
    if r.returncode != 0:
        pytest.skip("nvcc unavailable: " + r.stderr[-200:])
    out = subprocess.run([exe, "1000000"], capture_output=True, text=True, check=True).stdout
    n, badq, bade, maxulp = out.split()
    assert int(badq) == 0
    assert float(maxulp) <= 1.0
    assert int(bade) < int(n) // 100
