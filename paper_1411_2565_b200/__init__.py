"""Python binding of libgrace (include/grace.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``libgrace.so``; this
module converts numpy arrays / torch tensors to pointers and status codes to
exceptions.  There is no CPU fallback: if the library or a GPU is missing the
calls raise.

Functions keep the C names (``grace_create``, ``grace_set_m``, ...); ``Grace``
is a small object wrapper over them.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GRACE_LIB_PATH: an alternative in-tree build (tuning sweeps of compile-time knobs)
LIB_PATH = os.environ.get("GRACE_LIB_PATH") or os.path.join(_HERE, "libgrace.so")

GRACE_OK = 0
GRACE_EINVAL = -1
GRACE_ENOMEM = -2
GRACE_EZEROCELL = -3
GRACE_ENONFINITE = -4
GRACE_ECUDA = -5
GRACE_EUNSUPPORTED = -6
_NAMES = {-1: "EINVAL", -2: "ENOMEM", -3: "EZEROCELL", -4: "ENONFINITE", -5: "ECUDA", -6: "EUNSUPPORTED"}

# (name, restype, argtypes) of every symbol declared in include/grace.h
_D = ctypes.c_double
_I = ctypes.c_int
_P = ctypes.c_void_p
_PD = ctypes.POINTER(ctypes.c_double)
_PF = ctypes.POINTER(ctypes.c_float)
_PLL = ctypes.POINTER(ctypes.c_longlong)
SIGNATURES = [
    ("grace_create", _I, [_I, _I, _I, _D, _D, _D, _D, _D, _D, _D, _D, ctypes.POINTER(_P)]),
    ("grace_destroy", None, [_P]),
    ("grace_set_m", _I, [_P, _PD]),
    ("grace_get_m", _I, [_P, _PD]),
    ("grace_set_hext", _I, [_P, _D, _D, _D]),
    ("grace_heff", _I, [_P, _PD]),
    ("grace_step", _I, [_P, _I, _D]),
    ("grace_last_error", ctypes.c_char_p, []),
    ("grace_set_alpha", _I, [_P, _D]),
    ("grace_set_stream", _I, [_P, _P]),
    ("grace_set_m_device", _I, [_P, _P]),
    ("grace_get_m_device", _I, [_P, _P]),
    ("grace_mavg", _I, [_P, _PD]),
    ("grace_step_count", _I, [_P, _PLL]),
    ("grace_energy", _I, [_P, _PD]),
    ("grace_set_integrator", _I, [_P, _I]),
    ("grace_set_field_schedule", _I, [_P, _D, _D, _D, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong]),
    ("grace_max_torque", _I, [_P, _PD]),
    ("grace_relax", _I, [_P, _D, _D, ctypes.c_longlong, _D, _I, _PLL, _PD]),
    ("grace_last_nonfinite", _I, [_P, _PLL, _PLL]),
    ("grace_geometry", _I, [_P, _PLL]),
    ("grace_device_bytes", _I, [_P, ctypes.POINTER(ctypes.c_size_t)]),
    ("grace_tensor_octant", _I, [_I, _I, _I, _D, _D, _D, _PD]),
    ("grace_kernel_spectrum", _I, [_P, _PF]),
    ("grace_set_profiling", _I, [_P, _I]),
    ("grace_kernel_times", _I, [_P, _PD, _PLL, ctypes.POINTER(_I), _I]),
    ("grace_create_virtual", _I, [_I, _I, _I, _D, _D, _D, _D, _D, _D, _D, _D, _I, ctypes.POINTER(_P)]),
    ("grace_nccl_unique_id", _I, [_P]),
    ("grace_create_dist", _I, [_I, _I, _I, _D, _D, _D, _D, _D, _D, _D, _D, _I, _I, _P, ctypes.POINTER(_P)]),
    ("grace_partition", _I, [_P, _PLL]),
    ("grace_set_geometry", _I, [_P, _P]),
    ("grace_step_adaptive", _I, [_P, _D, _PD, _D, ctypes.c_longlong, _PLL, _PLL]),
    ("grace_kernel_spectrum_f64", _I, [_I, _I, _I, _D, _D, _D, _PD]),
    ("grace_set_m_f32", _I, [_P, _PF]),
    ("grace_get_m_f32", _I, [_P, _PF]),
]

_lib = None


class GraceError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"GRACE_{_NAMES.get(code, code)}: {msg}")
        self.code = code


def _torch_nccl():
    """torch's bundled libnccl (the NCCL torch.distributed uses), if installed."""
    try:
        import nvidia.nccl

        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return None


def load(path=LIB_PATH):
    """Load libgrace.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        # one NCCL per process: libgrace dlopens the library torch.distributed uses
        if "GRACE_NCCL_LIB" not in os.environ and _torch_nccl():
            os.environ["GRACE_NCCL_LIB"] = _torch_nccl()
        if not os.path.exists(path):
            raise ImportError(f"{path} not built; run __graft_entry__.build() (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(code):
    if code != GRACE_OK:
        raise GraceError(code, load().grace_last_error().decode())


def _f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} values, got {a.size}")
    return a


def _pd(a):
    return a.ctypes.data_as(_PD)


# ---- C-named functions -------------------------------------------------------

def grace_create(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma):
    h = _P()
    _check(load().grace_create(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, ctypes.byref(h)))
    return h


def grace_create_virtual(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, nranks):
    h = _P()
    _check(load().grace_create_virtual(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, nranks, ctypes.byref(h)))
    return h


def grace_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(load().grace_nccl_unique_id(buf))
    return bytes(buf.raw)


def grace_create_dist(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, rank, nranks, nccl_id):
    h = _P()
    idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
    _check(load().grace_create_dist(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, rank, nranks, idbuf,
                                    ctypes.byref(h)))
    return h


def grace_partition(h):
    out = (ctypes.c_longlong * 12)()
    _check(load().grace_partition(h, out))
    keys = ("P", "rank", "nz_local", "z_offset", "kx_block", "kx_columns", "pitch1", "pitch2", "pipelined",
            "graphs", "halo_comm", "p2p")
    return dict(zip(keys, list(out)))


def grace_destroy(h):
    load().grace_destroy(h)


def grace_set_m(h, m):
    m = _f64(m)
    _check(load().grace_set_m(h, _pd(m)))


def grace_get_m(h, out):
    _check(load().grace_get_m(h, _pd(out)))
    return out


def _pf(a):
    if a.dtype != np.float32 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous float32 array")
    return a.ctypes.data_as(_PF)


def grace_set_m_f32(h, m):
    """m: C-contiguous float32 [3][nz][ny][nx] host array (pinned for full PCIe speed)."""
    _check(load().grace_set_m_f32(h, _pf(m)))


def grace_get_m_f32(h, out):
    _check(load().grace_get_m_f32(h, _pf(out)))
    return out


def grace_set_hext(h, hx, hy, hz):
    _check(load().grace_set_hext(h, hx, hy, hz))


def grace_heff(h, out):
    _check(load().grace_heff(h, _pd(out)))
    return out


def grace_step(h, n, dt):
    _check(load().grace_step(h, int(n), float(dt)))


def grace_last_error():
    return load().grace_last_error().decode()


def grace_set_alpha(h, alpha):
    _check(load().grace_set_alpha(h, alpha))


def grace_set_geometry(h, mask_ptr):
    _check(load().grace_set_geometry(h, _P(mask_ptr) if mask_ptr else None))


def grace_set_stream(h, stream_ptr):
    _check(load().grace_set_stream(h, _P(stream_ptr) if stream_ptr else None))


def grace_set_m_device(h, dev_ptr):
    _check(load().grace_set_m_device(h, _P(dev_ptr)))


def grace_get_m_device(h, dev_ptr):
    _check(load().grace_get_m_device(h, _P(dev_ptr)))


def grace_mavg(h):
    out = np.zeros(3)
    _check(load().grace_mavg(h, _pd(out)))
    return out


def grace_set_field_schedule(h, h0, start, decay, stop):
    _check(load().grace_set_field_schedule(h, float(h0[0]), float(h0[1]), float(h0[2]), int(start), int(decay),
                                           int(stop)))


def grace_step_adaptive(h, t_span, dt, tol, max_attempts=10**9):
    """Advance t_span seconds with adaptive steps; returns (next dt, accepted, rejected)."""
    d = ctypes.c_double(dt)
    a, r = ctypes.c_longlong(0), ctypes.c_longlong(0)
    _check(load().grace_step_adaptive(h, t_span, ctypes.byref(d), tol, max_attempts, ctypes.byref(a),
                                      ctypes.byref(r)))
    return d.value, a.value, r.value


def grace_set_integrator(h, kind):
    _check(load().grace_set_integrator(h, {"euler": 0, "heun": 1}.get(kind, kind)))


def grace_energy(h):
    """(total, exchange, anisotropy, demag, zeeman) in joules."""
    out = (ctypes.c_double * 5)()
    _check(load().grace_energy(h, out))
    return tuple(out)


def grace_max_torque(h):
    v = ctypes.c_double()
    _check(load().grace_max_torque(h, ctypes.byref(v)))
    return v.value


def grace_relax(h, alpha_relax, dt, max_steps, tol, check_every):
    n, t = ctypes.c_longlong(), ctypes.c_double()
    _check(load().grace_relax(h, float(alpha_relax), float(dt), int(max_steps), float(tol), int(check_every),
                              ctypes.byref(n), ctypes.byref(t)))
    return n.value, t.value


def grace_step_count(h):
    v = ctypes.c_longlong()
    _check(load().grace_step_count(h, ctypes.byref(v)))
    return v.value


def grace_last_nonfinite(h):
    s, c = ctypes.c_longlong(), ctypes.c_longlong()
    _check(load().grace_last_nonfinite(h, ctypes.byref(s), ctypes.byref(c)))
    return s.value, c.value


def grace_geometry(h):
    out = (ctypes.c_longlong * 12)()
    _check(load().grace_geometry(h, out))
    keys = ("nx", "ny", "nz", "Px", "Py", "Pz", "Kx", "Kxp", "Kyh", "Kzh", "KSp", "kernels")
    return dict(zip(keys, list(out)))


def grace_device_bytes(h):
    v = ctypes.c_size_t()
    _check(load().grace_device_bytes(h, ctypes.byref(v)))
    return v.value


def grace_tensor_octant(nx, ny, nz, dx, dy, dz):
    out = np.empty((6, nz, ny, nx), dtype=np.float64)
    _check(load().grace_tensor_octant(nx, ny, nz, dx, dy, dz, _pd(out)))
    return out


def grace_kernel_spectrum(h):
    g = grace_geometry(h)
    out = np.empty((6, g["Kzh"], g["Kyh"], g["KSp"]), dtype=np.float32)
    _check(load().grace_kernel_spectrum(h, out.ctypes.data_as(_PF)))
    return out


def grace_kernel_spectrum_f64(nx, ny, nz, dx, dy, dz):
    """fp64 folded spectrum [6][Kzh][Kyh][KSp] before the fp32 rounding (standalone)."""
    def pad(n):
        if n == 1:
            return 1
        p = 1
        while p < 2 * n - 1:
            p <<= 1
        return p

    px, py, pz = pad(nx), pad(ny), pad(nz)
    kx = 1 if px == 1 else px // 2 + 1
    kyh = 1 if py == 1 else py // 2 + 1
    kzh = 1 if pz == 1 else pz // 2 + 1
    ksp = (kx + 31) // 32 * 32
    out = np.empty((6, kzh, kyh, ksp), dtype=np.float64)
    _check(load().grace_kernel_spectrum_f64(nx, ny, nz, dx, dy, dz, _pd(out)))
    return out


def grace_set_profiling(h, on):
    _check(load().grace_set_profiling(h, 1 if on else 0))


def grace_kernel_times(h, reset=False):
    cap = 8
    ms = (ctypes.c_double * cap)()
    ln = (ctypes.c_longlong * cap)()
    nk = ctypes.c_int(cap)
    _check(load().grace_kernel_times(h, ms, ln, ctypes.byref(nk), 1 if reset else 0))
    return list(ms)[: nk.value], list(ln)[: nk.value]


# ---- object wrapper ------------------------------------------------------------

class Grace:
    """One LLG context (owns its device memory).

    Default: the whole grid on the current GPU.  ``virtual_ranks=P`` partitions it
    into P z-slabs in this process (exchanges by device copies); ``dist=(rank,
    nranks, nccl_id)`` makes this process rank ``rank`` of an NCCL partition, and
    the arrays are then the local slab.
    """

    def __init__(self, n, d, Ms, A, Ku, alpha, gamma0, virtual_ranks=None, dist=None):
        self.n = tuple(int(v) for v in n)
        nz_here = self.n[2]
        if dist is not None:
            rank, nranks, nid = dist
            self.h = grace_create_dist(*self.n, *d, Ms, A, Ku, alpha, gamma0, rank, nranks, nid)
            nz_here = self.n[2] // nranks
        elif virtual_ranks is not None:
            self.h = grace_create_virtual(*self.n, *d, Ms, A, Ku, alpha, gamma0, int(virtual_ranks))
        else:
            self.h = grace_create(*self.n, *d, Ms, A, Ku, alpha, gamma0)
        self.shape = (3, nz_here, self.n[1], self.n[0])

    def close(self):
        if self.h:
            grace_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_m(self, M):
        grace_set_m(self.h, _f64(M, int(np.prod(self.shape))))

    def get_m(self):
        out = np.empty(self.shape)
        return grace_get_m(self.h, out)

    def set_hext(self, h):
        grace_set_hext(self.h, *[float(v) for v in h])

    def set_alpha(self, a):
        grace_set_alpha(self.h, float(a))

    def heff(self):
        out = np.empty(self.shape)
        return grace_heff(self.h, out)

    def step(self, n, dt):
        grace_step(self.h, n, dt)

    def mavg(self):
        return grace_mavg(self.h)

    @property
    def steps(self):
        return grace_step_count(self.h)

    @property
    def geometry(self):
        return grace_geometry(self.h)

    def set_field_schedule(self, h0, start, decay, stop):
        """Paper/SPEC field schedule: + a(k) h0 (A/m) on top of set_hext's field."""
        grace_set_field_schedule(self.h, h0, start, decay, stop)

    def set_geometry(self, mask):
        """Geometry mask uint8/bool [nz, ny, nx] (nonzero = magnetic; None removes it)."""
        if mask is None:
            grace_set_geometry(self.h, None)
            return
        m = np.ascontiguousarray(np.asarray(mask) != 0, dtype=np.uint8)
        if m.size != int(np.prod(self.shape[1:])):
            raise ValueError(f"mask of {m.size} cells for a grid of {int(np.prod(self.shape[1:]))}")
        grace_set_geometry(self.h, m.ctypes.data)

    def step_adaptive(self, t_span, dt, tol, max_attempts=10**9):
        return grace_step_adaptive(self.h, t_span, dt, tol, max_attempts)

    def set_integrator(self, kind):
        """'euler' (the paper's, default) or 'heun' (second order, two H_eff per step)."""
        grace_set_integrator(self.h, kind)

    def energy(self):
        """Eq. (1) energy terms in joules: dict total/exchange/anisotropy/demag/zeeman."""
        return dict(zip(("total", "exchange", "anisotropy", "demag", "zeeman"), grace_energy(self.h)))

    def max_torque(self):
        return grace_max_torque(self.h)

    def relax(self, alpha_relax=1.0, dt=1e-13, max_steps=1_000_000, tol=1e-4, check_every=100):
        """SPEC relax: returns (steps taken, final max torque)."""
        return grace_relax(self.h, alpha_relax, dt, max_steps, tol, check_every)
