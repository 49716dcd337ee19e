"""ctypes binding of the C ABI in include/finom_b200.h.

This is the only route to the numerics: there is no CPU fallback and no
backend switch.  If the shared library is missing or no CUDA device is
visible, every entry point raises DeviceError.
"""

import ctypes
import os

import numpy as np

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfinom_b200.so")
# The same sources built with 512-element tiles (16 merged elements per lane,
# 8 warps per SM): the tile-parallel loop of a few large problems runs faster
# on it (config 2: 2.19e10 vs 2.03e10 pts*it/s -- half the tiles, half the
# per-tile carry, record and reduction work), the group solve of batches and
# small problems on the 256-element tiles (config 5: 1040 vs 1209 ms per
# solve; config 1: 32.3 vs 33.5 us per iteration).  See lib_for().
LIB_T512_PATH = os.path.join(_HERE, "libfinom_b200_t512.so")
if os.environ.get("FINOM_LIB"):  # (A/B timing of a library variant built in-tree)
    LIB_PATH = os.path.abspath(os.environ["FINOM_LIB"])

_c_i64 = ctypes.c_int64
_c_dbl = ctypes.c_double
_c_int = ctypes.c_int
_vp = ctypes.c_void_p

# name -> (restype, argtypes); must match include/finom_b200.h
SIGNATURES = {
    "finom_last_error": (ctypes.c_char_p, []),
    "finom_build_info": (ctypes.c_char_p, []),
    "finom_plan1d_create": (_c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_plan1d_destroy": (_c_int, [_vp]),
    "finom_plan1d_create_v": (_c_int, [_c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_stage_pieces": (_c_int, [_c_int, _vp, _vp, _c_i64, _vp]),
    "finom_tile_partition": (_c_i64, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _vp]),
    "finom_plan1d_info": (_c_int, [_vp, _vp]),
    "finom_solve1d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int,
                               _c_dbl, _vp, _vp, _vp, _vp]),
    "finom_solve1d_async": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int,
                                     _c_dbl, _vp, _vp, _vp, _vp]),
    "finom_cost1d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_apply1d": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _vp, _vp, _vp]),
    "finom_iterate1d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_profile1d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_int, _c_dbl,
                                 _vp, _vp, _vp]),
    "finom_solve1d_launches": (_c_i64, [_vp, _c_i64, _c_int]),
    "finom_solve1d_group": (_c_int, [_vp]),
    "finom_stage_copy": (_c_int, [_c_int, _vp, _vp, _c_i64]),
    "finom_sinkhorn1d_host": (_c_int, [_c_i64, _vp, _c_i64, _vp, _vp, _vp, _c_dbl, _c_i64,
                                       _c_dbl, _c_int, _c_dbl, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _vp, _vp]),
    "finom_sinkhorn2d_host": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _vp,
                                       _vp, _c_dbl, _c_i64, _c_dbl, _c_int, _c_dbl, _vp, _vp,
                                       _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int]),
    "finom_apply2d_host": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_dbl,
                                    _vp, _vp, _vp, _c_int, _vp]),
    "finom_cost2d_host": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_dbl,
                                   _vp, _vp, _vp, _vp, _vp]),
    "finom_release_memory": (_c_int, []),
    "finom_dense1d": (_c_int, [_c_i64, _c_i64, _vp, _vp, _vp, _vp, _c_dbl, _vp, _vp, _vp, _vp]),
    "finom_dense2d": (_c_int, [_c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp,
                               _c_dbl, _vp, _vp, _vp, _vp]),
    "finom_grid_create": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _vp,
                                   _vp]),
    "finom_grid_destroy": (_c_int, [_vp]),
    "finom_grid_info": (_c_int, [_vp, _vp]),
    "finom_solve2d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int, _c_dbl,
                               _vp, _vp, _vp, _vp]),
    "finom_cost2d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_apply2d": (_c_int, [_vp, _vp, _vp, _c_int, _vp, _vp, _vp]),
    "finom_grid_set_shifts": (_c_int, [_vp, _vp, _vp, _vp]),
    "finom_iterate2d": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_seg1d_split": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp]),
    "finom_seg1d_create": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_dbl, _c_i64, _c_i64, _vp, _vp]),
    "finom_seg1d_destroy": (_c_int, [_vp]),
    "finom_seg1d_window": (_c_int, [_vp, _vp]),
    "finom_seg1d_pre": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "finom_seg1d_finish": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_seg1d_absorb": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_grid2d_create": (_c_int, [_c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_dbl, _c_i64,
                                     _c_i64, _vp]),
    "finom_grid2d_destroy": (_c_int, [_vp]),
    "finom_grid2d_set_shifts": (_c_int, [_vp, _vp, _vp, _vp]),
    "finom_grid2d_xpre": (_c_int, [_vp, _c_int, _vp, _vp, _c_int, _vp, _vp]),
    "finom_grid2d_finish": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_int,
                                     _vp, _vp, _vp, _vp]),
    "finom_grid2d_edges": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _vp, _vp]),
    "finom_grid2d_absorb_nb": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "finom_grid2d_decide": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int,
                                     _c_dbl, _vp]),
    "finom_seg1d_decide": (_c_int, [_vp, _vp, _c_int, _vp, _vp, _vp, _c_i64, _c_dbl, _c_int,
                                    _c_dbl, _vp]),
    "finom_grid2d_absorb": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                                     _vp]),
}

_lib = None


def load(require_device=True):
    """Load libfinom_b200.so (and check a CUDA device is present)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                "CUDA extension %s is not built; run __graft_entry__.build()" % LIB_PATH)
        _lib = _bind(ctypes.CDLL(LIB_PATH))
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible; the FINOM B200 path has no CPU fallback")
    return _lib


_lib_t512 = None


def _bind(lib):
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def use_t512(P, merged):
    """lib_for's rule (host only)."""
    want = os.environ.get("FINOM_TILE")
    return want == "512" or (want != "256" and P <= 4 and merged >= (1 << 20))


def lib_for(P, merged):
    """The library a plan of P problems with `merged` elements (sum of n + m)
    runs on: the 512-element-tile build for at most 4 problems of >= 2^20
    merged elements (the tile-parallel loop over the whole GPU), the default
    256-element build otherwise.  FINOM_TILE=256 / 512 forces one."""
    global _lib_t512
    if not use_t512(P, merged) or os.environ.get("FINOM_LIB"):
        return load()
    if _lib_t512 is None:
        load()  # (device check)
        if not os.path.exists(LIB_T512_PATH):
            raise DeviceError("CUDA extension %s is not built; run __graft_entry__.build()"
                              % LIB_T512_PATH)
        _lib_t512 = _bind(ctypes.CDLL(LIB_T512_PATH))
    return _lib_t512


def stage_copy(direction, host, dev):
    """Contiguous host numpy array <-> device tensor through the library's pinned
    staging (finom_stage_copy; direction 0: host -> device, 1: device -> host)."""
    assert host.flags["C_CONTIGUOUS"] and host.nbytes == dev.numel() * dev.element_size()
    check(load().finom_stage_copy(direction, ptr(host), ptr(dev), host.nbytes), "finom_stage_copy")


def stage_pieces(direction, hosts, dev):
    """List of contiguous host numpy arrays <-> one device tensor, in order
    (finom_stage_pieces; 0: gather into dev, 1: scatter into the arrays)."""
    hosts = list(hosts)
    assert all(h.flags["C_CONTIGUOUS"] for h in hosts)
    assert sum(h.nbytes for h in hosts) == dev.numel() * dev.element_size()
    hp = np.array([h.ctypes.data for h in hosts], dtype=np.uint64)
    nb = np.array([h.nbytes for h in hosts], dtype=np.int64)
    check(load().finom_stage_pieces(direction, ptr(hp), ptr(nb), len(hosts), ptr(dev)),
          "finom_stage_pieces")


def tile_partition(x, y):
    """Host-only tile partition + merged-order masks (finom_tile_partition)."""
    lib = load(require_device=False)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    T = lib.finom_tile_partition(x.size, ptr(x), y.size, ptr(y), 0, None, None)
    tiles = np.zeros((T, 4), dtype=np.int32)
    masks = np.zeros((T, 16), dtype=np.uint32)
    lib.finom_tile_partition(x.size, ptr(x), y.size, ptr(y), T, ptr(tiles), ptr(masks))
    return tiles, masks


def last_error():
    return load(False).finom_last_error().decode()


def ptr(a):
    """Raw pointer of a numpy array or a torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


def check(code, what, lib=None):
    """Map a C status >= 100 to DeviceError; return FINOM status 0/1/2.
    (lib: the library the call went to, for its error message.)"""
    if code >= 100:
        msg = (lib or load(False)).finom_last_error().decode()
        raise DeviceError("%s failed: %s" % (what, msg))
    return code


class Plan1D:
    """Device plan for a batch of P 1D problems (finom_plan1d_create)."""

    def __init__(self, xs, ys, eps):
        xs = [np.ascontiguousarray(x, dtype=np.float64) for x in xs]
        ys = [np.ascontiguousarray(y, dtype=np.float64) for y in ys]
        lib = lib_for(len(xs), sum(x.size for x in xs) + sum(y.size for y in ys))
        self.P = len(xs)
        self.xoff = np.zeros(self.P + 1, dtype=np.int64)
        self.yoff = np.zeros(self.P + 1, dtype=np.int64)
        self.xoff[1:] = np.cumsum([x.size for x in xs])
        self.yoff[1:] = np.cumsum([y.size for y in ys])
        self.eps = np.ascontiguousarray(np.broadcast_to(np.asarray(eps, dtype=np.float64),
                                                        (self.P,)))
        h = ctypes.c_void_p()
        if self.P == 1:
            check(lib.finom_plan1d_create(1, ptr(self.xoff), ptr(xs[0]), ptr(self.yoff),
                                          ptr(ys[0]), ptr(self.eps), stream_ptr(),
                                          ctypes.byref(h)), "finom_plan1d_create", lib)
        else:  # per-problem arrays staged as they are (no host concatenation)
            n = np.diff(self.xoff)
            m = np.diff(self.yoff)
            xp = np.array([x.ctypes.data for x in xs], dtype=np.uint64)
            yp = np.array([y.ctypes.data for y in ys], dtype=np.uint64)
            check(lib.finom_plan1d_create_v(self.P, ptr(n), ptr(xp), ptr(m), ptr(yp),
                                            ptr(self.eps), stream_ptr(), ctypes.byref(h)),
                  "finom_plan1d_create_v", lib)
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    @property
    def lib(self):
        """The library the plan lives in (every call on the handle goes there)."""
        return self._lib

    def info(self):
        out = np.zeros(8, dtype=np.int64)
        check(self._lib.finom_plan1d_info(self._h, ptr(out)), "finom_plan1d_info", self._lib)
        keys = ("P", "tiles", "NX", "NY", "max_tiles", "tile", "threads", "smem")
        return dict(zip(keys, (int(v) for v in out)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.finom_plan1d_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Grid:
    """Device plan of a 2D grid pair (finom_grid_create): sweep plans, scratch
    grids and solve state, reused by every solve / iterate / cost / apply."""

    def __init__(self, x1, y1, x2, y2, eps):
        lib = load()
        self._mesh = [np.ascontiguousarray(z, dtype=np.float64) for z in (x1, y1, x2, y2)]
        x1, y1, x2, y2 = self._mesh
        self.shape_u = (x1.size, y1.size)
        self.shape_v = (x2.size, y2.size)
        self.eps = float(eps)
        h = ctypes.c_void_p()
        check(lib.finom_grid_create(x1.size, ptr(x1), y1.size, ptr(y1), x2.size, ptr(x2),
                                    y2.size, ptr(y2), self.eps, stream_ptr(), ctypes.byref(h)),
              "finom_grid_create")
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def info(self):
        out = np.zeros(8, dtype=np.int64)
        check(self._lib.finom_grid_info(self._h, ptr(out)), "finom_grid_info")
        keys = ("n1", "m1", "n2", "m2", "tables", "square_x", "square_y", "launches")
        return dict(zip(keys, (int(v) for v in out)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.finom_grid_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev(a):
    import torch
    return None if a is None else torch.from_numpy(np.array(a, dtype=np.float64)).cuda()


def dense1d(x, y, a, b, eps, phi=None, psi=None):
    """Dense kernel (or plan with phi / psi) of a 1D pair on the device
    (finom_dense1d); returns a host n x m array."""
    import torch
    n, m = len(x), len(y)
    args = [_dev(z) for z in (x, y, a, b, phi, psi)]
    out = torch.empty(n * m, dtype=torch.float64, device="cuda")
    check(load().finom_dense1d(n, m, *(ptr(z) for z in args[:4]), float(eps),
                               ptr(args[4]), ptr(args[5]), ptr(out), stream_ptr()),
          "finom_dense1d")
    return out.cpu().numpy().reshape(n, m)


def dense2d(x1, y1, x2, y2, A, B, eps, phi=None, psi=None):
    """Dense kernel (or plan) of a grid pair on the device (finom_dense2d)."""
    import torch
    n1, m1, n2, m2 = len(x1), len(y1), len(x2), len(y2)
    args = [_dev(z) for z in (x1, y1, x2, y2, A, B, phi, psi)]
    out = torch.empty(n1 * m1 * n2 * m2, dtype=torch.float64, device="cuda")
    check(load().finom_dense2d(n1, m1, n2, m2, *(ptr(z) for z in args[:6]), float(eps),
                               ptr(args[6]), ptr(args[7]), ptr(out), stream_ptr()),
          "finom_dense2d")
    return out.cpu().numpy().reshape(n1 * m1, n2 * m2)
