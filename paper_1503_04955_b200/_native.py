"""ctypes binding of libdkss.so (include/dkss.h).

The library is built in-tree (``python -m paper_1503_04955_b200.build``) into
``paper_1503_04955_b200/_lib/libdkss.so``.  There is no CPU fallback: if the
library is missing or cannot be loaded, every GPU entry point raises
``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DKSS_LIB") or os.path.join(HERE, "_lib", "libdkss.so")

# every symbol include/dkss.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "dkss_plan_create", "dkss_plan_create_ex", "dkss_plan_destroy", "dkss_plan_get_info", "dkss_last_error",
    "dkss_version", "dkss_kernel_launches", "dkss_footprint_bytes", "dkss_host_alloc", "dkss_host_free",
    "dkss_mul", "dkss_mul_digits", "dkss_mul_batch_digits", "dkss_mul_batch", "dkss_mul_device", "dkss_profile_device",
    "dkss_encode_host", "dkss_fft_host", "dkss_rmul_host", "dkss_decode_host",
    "dkss_fs_layout_get", "dkss_fs_columns_fwd", "dkss_fs_rows", "dkss_fs_columns_inv",
    "dkss_block_transpose", "dkss_decode_device", "dkss_lucas_lehmer", "dkss_fs_decode_partial",
    "dkss_fs_decode_finish", "dkss_fs_columns_fwd_peer", "dkss_fs_rows_peer", "dkss_ipc_alloc", "dkss_ipc_open",
    "dkss_ipc_close", "dkss_ipc_free",
    # include/smul.h
    "smul_plan_create", "smul_plan_destroy", "smul_product_limbs", "smul_mul", "smul_mul_digits", "smul_mul_device",
    "smul_fft_host",
)

DKSS_OK, DKSS_EINVAL, DKSS_ECUDA, DKSS_ERANGE, DKSS_ENOMEM = 0, -1, -2, -3, -4
DKSS_DIGITS_TRUSTED = 0x100  # digit_bits flag: digits already known to fit (include/dkss.h)
# dkss_plan_opts values (include/dkss.h)
ROW_PHASES = {"auto": 0, "launches": 1, "persistent": 2, "cluster": 3}
PASS_KINDS = {"auto": 0, "cta": 1, "warp": 2, "split": 3}
TWIDDLE_ENGINES = {"auto": 0, "cuda": 1, "tensor": 2}


class NativeUnavailable(RuntimeError):
    pass


class DkssError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libdkss error {code}: {msg}")
        self.code = code


class PlanDesc(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("M", ctypes.c_int32), ("m", ctypes.c_int32), ("u", ctypes.c_int32),
                ("L", ctypes.c_int32), ("p", ctypes.POINTER(ctypes.c_uint32)),
                ("rho_powers", ctypes.POINTER(ctypes.c_uint32))]


class PlanInfo(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("M", ctypes.c_int32), ("m", ctypes.c_int32), ("u", ctypes.c_int32),
                ("L", ctypes.c_int32), ("levels", ctypes.c_int32), ("base_len", ctypes.c_int32),
                ("poly_bytes", ctypes.c_int64), ("operand_limbs", ctypes.c_int64),
                ("product_limbs", ctypes.c_int64), ("ring_products", ctypes.c_int64),
                ("twiddles_per_fft", ctypes.c_int64), ("launches_per_mul", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_int64), ("footprint_bytes", ctypes.c_int64)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("row_phase", ctypes.c_int32), ("pass_kind", ctypes.c_int32), ("twiddle", ctypes.c_int32)]


class FsLayout(ctypes.Structure):
    _fields_ = [("cols", ctypes.c_int64), ("rows", ctypes.c_int64), ("elem_words", ctypes.c_int64),
                ("block_words", ctypes.c_int64), ("decode_seg", ctypes.c_int64)]


class SmulPlanDesc(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("m", ctypes.c_int32), ("s", ctypes.c_int64), ("K", ctypes.c_int32),
                ("omega_exp", ctypes.c_int32)]


_u32p = ctypes.POINTER(ctypes.c_uint32)
_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load libdkss.so (raises NativeUnavailable, never falls back)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} is missing: run `python -m paper_1503_04955_b200.build`")
        try:
            L = ctypes.CDLL(path)
        except OSError as e:
            raise NativeUnavailable(f"cannot load {path}: {e}") from e
        vp = ctypes.c_void_p
        L.dkss_plan_create.argtypes = [ctypes.POINTER(PlanDesc), ctypes.c_int, ctypes.POINTER(vp)]
        L.dkss_plan_create_ex.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(PlanOpts), ctypes.c_int,
                                          ctypes.POINTER(vp)]
        L.dkss_kernel_launches.restype = ctypes.c_int64
        L.dkss_kernel_launches.argtypes = []
        L.dkss_footprint_bytes.restype = ctypes.c_int64
        L.dkss_footprint_bytes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.dkss_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(vp)]
        L.dkss_host_free.argtypes = [vp]
        L.dkss_host_free.restype = None
        L.dkss_plan_destroy.argtypes = [vp]
        L.dkss_plan_destroy.restype = None
        L.dkss_plan_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.dkss_last_error.restype = ctypes.c_char_p
        L.dkss_mul.argtypes = [vp, _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t]
        L.dkss_mul_digits.argtypes = [vp, vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_int, _u32p,
                                      ctypes.c_size_t]
        L.dkss_mul_batch_digits.argtypes = [vp, ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t), ctypes.c_int, _u32p,
                                            ctypes.c_size_t]
        L.dkss_mul_batch.argtypes = [vp, ctypes.c_int, _u32p, _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t]
        L.dkss_mul_device.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_size_t, vp, ctypes.c_size_t, vp]
        L.dkss_profile_device.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_size_t, vp, vp, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_float),
                                          ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int)]
        L.dkss_encode_host.argtypes = [vp, _u32p, ctypes.c_size_t, _u32p]
        L.dkss_fft_host.argtypes = [vp, _u32p, ctypes.c_int]
        L.dkss_rmul_host.argtypes = [vp, _u32p, _u32p, _u32p, ctypes.c_size_t]
        L.dkss_decode_host.argtypes = [vp, _u32p, _u32p, ctypes.c_size_t]
        L.dkss_fs_layout_get.argtypes = [vp, ctypes.c_int, ctypes.POINTER(FsLayout)]
        L.dkss_fs_columns_fwd.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp, vp]
        L.dkss_fs_rows.argtypes = [vp, ctypes.c_int, vp, vp]
        L.dkss_fs_columns_inv.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp]
        L.dkss_fs_columns_fwd_peer.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t, vp, vp, vp]
        L.dkss_fs_rows_peer.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.dkss_ipc_alloc.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(vp), vp]
        L.dkss_ipc_open.argtypes = [ctypes.c_int, vp, ctypes.POINTER(vp)]
        L.dkss_ipc_close.argtypes = [vp]
        L.dkss_ipc_free.argtypes = [vp]
        L.dkss_block_transpose.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp]
        L.dkss_decode_device.argtypes = [vp, vp, vp, ctypes.c_size_t, vp]
        L.dkss_fs_decode_partial.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.dkss_fs_decode_finish.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_size_t, vp]
        L.dkss_lucas_lehmer.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, _u32p, ctypes.c_size_t]
        L.smul_plan_create.argtypes = [ctypes.POINTER(SmulPlanDesc), ctypes.c_int, ctypes.POINTER(vp)]
        L.smul_plan_destroy.argtypes = [vp]
        L.smul_plan_destroy.restype = None
        L.smul_product_limbs.argtypes = [vp]
        L.smul_product_limbs.restype = ctypes.c_int64
        L.smul_mul.argtypes = [vp, _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t, _u32p, ctypes.c_size_t]
        L.smul_mul_device.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_size_t, vp, ctypes.c_size_t, vp]
        L.smul_mul_digits.argtypes = [vp, vp, ctypes.c_size_t, vp, ctypes.c_size_t, ctypes.c_int, _u32p, ctypes.c_size_t]
        L.smul_fft_host.argtypes = [vp, _u32p, _u32p, ctypes.c_int]
        for name in EXPORTS:
            if not hasattr(L, name):
                raise NativeUnavailable(f"{path} lacks symbol {name}")
        _lib = L
        return L


def _ptr(a: np.ndarray):
    if a.dtype != np.uint32 or not a.flags.c_contiguous:
        raise TypeError("expected a C-contiguous uint32 array")
    return a.ctypes.data_as(_u32p)


def _check(rc: int):
    if rc != DKSS_OK:
        msg = load().dkss_last_error().decode(errors="replace")
        if rc in (DKSS_EINVAL, DKSS_ERANGE):
            raise ValueError(f"libdkss: {msg}")
        raise DkssError(rc, msg)


class DevicePlan:
    """A plan uploaded to one GPU (twiddle table in Montgomery form + workspace)."""

    def __init__(self, N: int, M: int, m: int, u: int, p: int, rho_powers, device: int = 0,
                 row_phase: str = "auto", pass_kind: str = "auto", twiddle: str = "auto"):
        """row_phase / pass_kind / twiddle pick a kernel shape (include/dkss.h dkss_plan_opts);
        "auto" is the measured-fastest one for the plan, the others exist so every variant can be
        tested (twiddle: "cuda" = IMAD.WIDE ring products, "tensor" = tcgen05 kind::i8)."""
        lib = load()
        self.N, self.M, self.m, self.u, self.p, self.device = N, M, m, u, p, device
        self.L = L = -(-p.bit_length() // 32)
        p_l = np.frombuffer(p.to_bytes(4 * L, "little"), dtype=np.uint32).copy()
        raw = b"".join(c.to_bytes(4 * L, "little") for row in rho_powers for c in row)
        rho_l = np.frombuffer(raw, dtype=np.uint32).copy()
        desc = PlanDesc(N, M, m, u, L, _ptr(p_l), _ptr(rho_l))
        h = ctypes.c_void_p()
        opts = PlanOpts(ROW_PHASES[row_phase], PASS_KINDS[pass_kind], TWIDDLE_ENGINES[twiddle])
        _check(lib.dkss_plan_create_ex(ctypes.byref(desc), ctypes.byref(opts), device, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.info = self.get_info()

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.dkss_plan_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def handle(self):
        return self._h

    def get_info(self) -> dict:
        info = PlanInfo()
        _check(self._lib.dkss_plan_get_info(self._h, ctypes.byref(info)))
        return {k: getattr(info, k) for k, _ in PlanInfo._fields_}

    @property
    def poly_shape(self):
        return (2 * self.M, self.m, self.L)

    # -- products --------------------------------------------------------------
    def mul_limbs(self, a: np.ndarray, b: np.ndarray, nc: int) -> np.ndarray:
        out = np.zeros(nc, dtype=np.uint32)
        _check(self._lib.dkss_mul(self._h, _ptr(a), a.size, _ptr(b), b.size, _ptr(out), nc))
        return out

    def mul_digits(self, a_ptr: int, na: int, b_ptr: int, nb: int, digit_bits: int, nc: int) -> np.ndarray:
        """Product of two radix-2^digit_bits digit strings at host addresses a_ptr / b_ptr."""
        out = pinned_empty((nc,))
        _check(self._lib.dkss_mul_digits(self._h, ctypes.c_void_p(a_ptr), na, ctypes.c_void_p(b_ptr), nb, digit_bits,
                                         _ptr(out), nc))
        return out

    def mul_batch_digits(self, a_ptrs, na, b_ptrs, nb, digit_bits: int, nc: int, out=None) -> np.ndarray:
        """Products of pairs of radix-2^digit_bits digit strings (host addresses + counts);
        `out`, if given, is a C-contiguous uint32[batch][nc] the products are written to."""
        batch = len(a_ptrs)
        vpa = (ctypes.c_void_p * batch)(*a_ptrs)
        vpb = (ctypes.c_void_p * batch)(*b_ptrs)
        cna = (ctypes.c_size_t * batch)(*na)
        cnb = (ctypes.c_size_t * batch)(*nb)
        if out is None:
            out = pinned_empty((batch, nc))
        elif out.shape != (batch, nc) or out.dtype != np.uint32 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous uint32[batch][nc] array")
        _check(self._lib.dkss_mul_batch_digits(self._h, batch, vpa, cna, vpb, cnb, digit_bits, _ptr(out), nc))
        return out

    def mul_batch(self, a: np.ndarray, b: np.ndarray, nc: int | None = None) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        batch, nl = a.shape
        nc = nc or self.info["product_limbs"]
        out = np.zeros((batch, nc), dtype=np.uint32)
        _check(self._lib.dkss_mul_batch(self._h, batch, _ptr(a), _ptr(b), nl, _ptr(out), nc))
        return out

    def mul_device(self, batch: int, a_ptr: int, b_ptr: int, n_limbs: int, c_ptr: int, nc: int, stream: int = 0):
        _check(self._lib.dkss_mul_device(self._h, batch, ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), n_limbs,
                                         ctypes.c_void_p(c_ptr), nc, ctypes.c_void_p(stream)))

    KIND_NAMES = {0: "encode", 1: "fwd_pass", 2: "bottom", 3: "inv_pass", 4: "decode1", 5: "decode2", 8: "twiddle_tc",
                  6: "transpose", 7: "rows"}

    def profile_device(self, batch: int, a_ptr: int, b_ptr: int, n_limbs: int, c_ptr: int, stream: int = 0):
        """Per-launch (kind, ms, limb-products, bytes) of one multiply, timed with CUDA events."""
        mx = 64
        kinds = (ctypes.c_int32 * mx)()
        ms = (ctypes.c_float * mx)()
        work = (ctypes.c_int64 * mx)()
        nbytes = (ctypes.c_int64 * mx)()
        n = ctypes.c_int()
        _check(self._lib.dkss_profile_device(self._h, batch, ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr), n_limbs,
                                             ctypes.c_void_p(c_ptr), ctypes.c_void_p(stream), mx, kinds, ms, work,
                                             nbytes, ctypes.byref(n)))
        return [(self.KIND_NAMES[kinds[i]], ms[i], work[i], nbytes[i]) for i in range(n.value)]

    # -- stages ----------------------------------------------------------------
    def encode(self, a_limbs: np.ndarray) -> np.ndarray:
        out = np.zeros(self.poly_shape, dtype=np.uint32)
        _check(self._lib.dkss_encode_host(self._h, _ptr(a_limbs), a_limbs.size, _ptr(out)))
        return out

    def fft(self, polys: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(polys, dtype=np.uint32).copy()
        count = v.size // (2 * self.M * self.m * self.L)
        _check(self._lib.dkss_fft_host(self._h, _ptr(v), count))
        return v

    def rmul(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.ascontiguousarray(y, dtype=np.uint32)
        out = np.empty_like(x)
        count = x.size // (self.m * self.L)
        _check(self._lib.dkss_rmul_host(self._h, _ptr(x), _ptr(y), _ptr(out), count))
        return out

    def decode(self, v: np.ndarray, nout: int) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.uint32)
        out = np.zeros(nout, dtype=np.uint32)
        _check(self._lib.dkss_decode_host(self._h, _ptr(v), _ptr(out), nout))
        return out

    # -- four-step split (device pointers, stream-ordered; see include/dkss.h) ----
    def fs_layout(self, world: int) -> dict:
        lay = FsLayout()
        _check(self._lib.dkss_fs_layout_get(self._h, world, ctypes.byref(lay)))
        return {k: getattr(lay, k) for k, _ in FsLayout._fields_}

    def fs_columns_fwd(self, rank: int, world: int, a_ptr: int, b_ptr: int, n_limbs: int, x_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_columns_fwd(self._h, rank, world, ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr),
                                             n_limbs, ctypes.c_void_p(x_ptr), ctypes.c_void_p(stream)))

    def fs_rows(self, world: int, z_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_rows(self._h, world, ctypes.c_void_p(z_ptr), ctypes.c_void_p(stream)))

    def fs_columns_fwd_peer(self, rank: int, world: int, a_ptr: int, b_ptr: int, n_limbs: int, x_ptr: int,
                            z_peers_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_columns_fwd_peer(self._h, rank, world, ctypes.c_void_p(a_ptr), ctypes.c_void_p(b_ptr),
                                                  n_limbs, ctypes.c_void_p(x_ptr), ctypes.c_void_p(z_peers_ptr),
                                                  ctypes.c_void_p(stream)))

    def fs_rows_peer(self, rank: int, world: int, z_ptr: int, x_peers_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_rows_peer(self._h, rank, world, ctypes.c_void_p(z_ptr), ctypes.c_void_p(x_peers_ptr),
                                           ctypes.c_void_p(stream)))

    def fs_columns_inv(self, rank: int, world: int, x_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_columns_inv(self._h, rank, world, ctypes.c_void_p(x_ptr), ctypes.c_void_p(stream)))

    def block_transpose(self, src_ptr: int, dst_ptr: int, n: int, a: int, b: int, run_words: int, stream: int = 0):
        _check(self._lib.dkss_block_transpose(self._h, ctypes.c_void_p(src_ptr), ctypes.c_void_p(dst_ptr), n, a, b,
                                              run_words, ctypes.c_void_p(stream)))

    def fs_decode_partial(self, rank: int, world: int, x_ptr: int, s_ptr: int, stream: int = 0):
        _check(self._lib.dkss_fs_decode_partial(self._h, rank, world, ctypes.c_void_p(x_ptr), ctypes.c_void_p(s_ptr),
                                                ctypes.c_void_p(stream)))

    def fs_decode_finish(self, world: int, parts_ptr: int, out_ptr: int, nc: int, stream: int = 0):
        _check(self._lib.dkss_fs_decode_finish(self._h, world, ctypes.c_void_p(parts_ptr), ctypes.c_void_p(out_ptr), nc,
                                               ctypes.c_void_p(stream)))

    def decode_device(self, v_ptr: int, out_ptr: int, nc: int, stream: int = 0):
        _check(self._lib.dkss_decode_device(self._h, ctypes.c_void_p(v_ptr), ctypes.c_void_p(out_ptr), nc,
                                            ctypes.c_void_p(stream)))

    def lucas_lehmer(self, p: int, iters: int, s: np.ndarray) -> np.ndarray:
        """`iters` Lucas-Lehmer steps s <- s^2 - 2 mod 2^p - 1 on the device (s: u32 limbs)."""
        s = np.ascontiguousarray(s, dtype=np.uint32).copy()
        _check(self._lib.dkss_lucas_lehmer(self._h, p, iters, _ptr(s), s.size))
        return s


class SmulDevicePlan:
    """An outermost Schoenhage-Strassen plan (bigmul/smul.py:20-30) on one GPU (include/smul.h)."""

    def __init__(self, N: int, m: int, s: int, K: int, omega_exp: int, device: int = 0):
        lib = load()
        self.N, self.m, self.s, self.K, self.omega_exp, self.device = N, m, s, K, omega_exp, device
        desc = SmulPlanDesc(N, m, s, K, omega_exp)
        h = ctypes.c_void_p()
        _check(lib.smul_plan_create(ctypes.byref(desc), device, ctypes.byref(h)))
        self._h = h
        self._lib = lib
        self.product_limbs = int(lib.smul_product_limbs(h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.smul_plan_destroy(self._h)
            self._h = None

    __del__ = close

    def mul_limbs(self, a: np.ndarray, b: np.ndarray, nc: int) -> np.ndarray:
        out = np.zeros(max(nc, 1), dtype=np.uint32)
        if b is a:
            _check(self._lib.smul_mul(self._h, _ptr(a), a.size, _ptr(a), a.size, _ptr(out), nc))
        else:
            _check(self._lib.smul_mul(self._h, _ptr(a), a.size, _ptr(b), b.size, _ptr(out), nc))
        return out[:nc]

    def mul_digits(self, a_ptr: int, na: int, b_ptr: int, nb: int, digit_bits: int, nc: int) -> np.ndarray:
        """Product of two radix-2^digit_bits digit strings (host addresses + counts)."""
        out = np.zeros(max(nc, 1), dtype=np.uint32)
        _check(self._lib.smul_mul_digits(self._h, a_ptr, na, b_ptr, nb, digit_bits, _ptr(out), nc))
        return out[:nc]

    def mul_device(self, batch: int, a_ptr: int, b_ptr: int, n_limbs: int, c_ptr: int, nc: int, stream: int = 0):
        _check(self._lib.smul_mul_device(self._h, batch, a_ptr, b_ptr, n_limbs, c_ptr, nc, stream))

    def fft(self, x: np.ndarray, top: np.ndarray, inverse: bool = False):
        """fft_eval in place: x uint32[n][K/32], top uint32[n]; shuffled in, natural out."""
        _check(self._lib.smul_fft_host(self._h, _ptr(x), _ptr(top), 1 if inverse else 0))


def kernel_launches() -> int:
    """Kernels launched through libdkss by this process so far (graph replays count each kernel
    node; include/dkss.h dkss_kernel_launches)."""
    return int(load().dkss_kernel_launches())


def footprint_bytes(N: int, M: int, m: int, L: int) -> int:
    """Device bytes one multiply of host operands holds for a plan of this shape
    (include/dkss.h dkss_footprint_bytes; no GPU needed)."""
    v = int(load().dkss_footprint_bytes(N, M, m, L))
    if v < 0:
        raise ValueError("bad plan shape")
    return v


_PINNED_MIN_BYTES = 64 << 10  # smaller products: ordinary memory (the staging copy is negligible)


class _PinnedBlock:
    """A page-locked block from the library pool (dkss_host_alloc), exposed to numpy through the
    array interface; numpy arrays (and their slices) built on it keep it alive, and the last one
    returns it to the pool."""

    __slots__ = ("ptr", "__array_interface__", "_free")

    def __init__(self, shape):
        lib = load()
        nbytes = 4 * int(np.prod(shape))
        p = ctypes.c_void_p()
        _check(lib.dkss_host_alloc(nbytes, ctypes.byref(p)))
        self.ptr = p.value
        self._free = lib.dkss_host_free
        self.__array_interface__ = {"shape": tuple(shape), "typestr": "<u4", "data": (self.ptr, False), "version": 3}

    def __del__(self):
        if self.ptr:
            self._free(ctypes.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(shape) -> np.ndarray:
    """uint32 array of `shape` in page-locked host memory for products (the device copies into it
    directly); below 64 KiB an ordinary array."""
    shape = tuple(shape)
    if 4 * int(np.prod(shape)) < _PINNED_MIN_BYTES:
        return np.empty(shape, dtype=np.uint32)
    return np.asarray(_PinnedBlock(shape))


IPC_HANDLE_BYTES = 64  # sizeof(cudaIpcMemHandle_t)


class IpcBuffer:
    """A device buffer other processes can map (dkss_ipc_alloc): `ptr`, `nbytes`, `handle` (bytes)."""

    def __init__(self, device: int, nbytes: int):
        L = load()
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(L.dkss_ipc_alloc(device, nbytes, ctypes.byref(p), h))
        self.ptr, self.nbytes, self.handle = p.value, nbytes, h.raw

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.dkss_ipc_free(ctypes.c_void_p(self.ptr))
            self.ptr = None


class IpcMapping:
    """Another process's IpcBuffer mapped into this one (dkss_ipc_open): `ptr`."""

    def __init__(self, device: int, handle: bytes):
        L = load()
        p = ctypes.c_void_p()
        _check(L.dkss_ipc_open(device, ctypes.create_string_buffer(handle, IPC_HANDLE_BYTES), ctypes.byref(p)))
        self.ptr = p.value

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.dkss_ipc_close(ctypes.c_void_p(self.ptr))
            self.ptr = None
