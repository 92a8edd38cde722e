"""B200-native randomized SVD (arXiv 1608.02148, the `rsvd` package) -- Python binding.

Thin ctypes binding of the C ABI in ``include/rsvd_b200.h``: argument
marshalling only.  Every step of the hot path (Omega, the passes over A, the
panel orthonormalisations, the Jacobi SVD, the IALM updates) runs in the CUDA
kernels of ``csrc/``; torch is used for device memory, streams and process
groups.  There is no CPU fallback: if the extension is missing this module
raises on import of the library.

Paper interfaces mirrored:
  rsvd(A, k, nu=NULL, nv=NULL, p=10, q=2, sdist="normal")     P:708   (§3.6)
  rpca(A, k, center=TRUE, scale=TRUE, retx=TRUE, p=10, q=2)   P:1381  (§4.4)
  predict(rpca object, newdata)
  rrpca(A, lambda=NULL, maxiter=50, tol=1e-5, p=10, q=2, ...) P:1736  (§5.4)
  rqb(A, k, p, q)                                             Alg. 4
  rid / rcur

The library's calls only enqueue work on the context's stream; every wrapper
here calls ``rsvd_sync`` afterwards (and raises on a numerical failure)
unless ``sync=False`` is passed, in which case ``Context.sync()`` reports it.
"""
import threading
import ctypes
import os
from collections import namedtuple

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "librsvd_b200.so")

SDIST = {"normal": 0, "unif": 1, "rademacher": 2}
STATUS = {0: "RSVD_OK", 1: "RSVD_EINVAL", 2: "RSVD_ENOMEM", 3: "RSVD_ECUDA", 4: "RSVD_ENCCL",
          5: "RSVD_ENUMERIC", 6: "RSVD_EUNSUPPORTED"}
EXPORTS = ["rsvd_create", "rsvd_destroy", "rsvd_last_error", "rsvd_version", "rsvd_sync", "rsvd_nccl_unique_id",
           "rsvd_comm_init", "rsvd_group_create", "rsvd_group_destroy", "rsvd_comm_init_group",
           "rsvd_params_default", "rsvd_workspace_bytes", "rsvd_run", "rsvd_run_host", "rsvd_rqb",
           "rsvd_rpca_params_default", "rsvd_rpca", "rsvd_rpca_host", "rsvd_rpca_predict",
           "rsvd_rrpca_params_default", "rsvd_rrpca", "rsvd_rrpca_host", "rsvd_omega", "rsvd_set_profiling", "rsvd_profile",
           "rsvd_profile_reset", "rsvd_launch_count", "rsvd_stats", "rsvd_rid", "rsvd_rcur"]


class RsvdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class Matrix(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("A", ctypes.c_void_p), ("m_local", ctypes.c_int64),
                ("n", ctypes.c_int64), ("lda", ctypes.c_int64), ("m_global", ctypes.c_int64),
                ("row_offset", ctypes.c_int64)]


class Params(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("nu", ctypes.c_int32), ("nv", ctypes.c_int32), ("p", ctypes.c_int32),
                ("q", ctypes.c_int32), ("sdist", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("stream", ctypes.c_uint64), ("center", ctypes.c_int32), ("scale", ctypes.c_int32),
                ("power", ctypes.c_int32)]

POWER = {"subspace": 0, "direct": 1, "lu": 2}


class PcaOut(ctypes.Structure):
    _fields_ = [("rotation", ctypes.c_void_p), ("ldr", ctypes.c_int64), ("eigvals", ctypes.c_void_p),
                ("sdev", ctypes.c_void_p), ("x", ctypes.c_void_p), ("ldx", ctypes.c_int64),
                ("center", ctypes.c_void_p), ("scale", ctypes.c_void_p), ("loadings", ctypes.c_void_p),
                ("ldl", ctypes.c_int64), ("x_white", ctypes.c_void_p), ("ldw", ctypes.c_int64),
                ("var_ratio", ctypes.c_void_p), ("var_cum", ctypes.c_void_p), ("total_var", ctypes.c_void_p)]


class RrpcaParams(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("tol", ctypes.c_double), ("maxiter", ctypes.c_int32),
                ("k", ctypes.c_int32), ("p", ctypes.c_int32), ("q", ctypes.c_int32), ("sdist", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("rand", ctypes.c_int32)]


_lib = None


def lib():
    """Load the C-ABI library (built in-tree by build.py).  Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("rsvd_b200 CUDA extension not built (%s); run __graft_entry__.build()" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    MP, PP = ctypes.POINTER(Matrix), ctypes.POINTER(Params)
    sig = {
        "rsvd_create": ([ctypes.POINTER(vp), ctypes.c_int, vp], ctypes.c_int),
        "rsvd_destroy": ([vp], ctypes.c_int),
        "rsvd_last_error": ([vp], ctypes.c_char_p),
        "rsvd_version": ([], ctypes.c_char_p),
        "rsvd_sync": ([vp], ctypes.c_int),
        "rsvd_nccl_unique_id": ([vp], ctypes.c_int),
        "rsvd_comm_init": ([vp, vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "rsvd_group_create": ([ctypes.POINTER(vp), ctypes.c_int], ctypes.c_int),
        "rsvd_group_destroy": ([vp], ctypes.c_int),
        "rsvd_comm_init_group": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "rsvd_params_default": ([PP, i32], None),
        "rsvd_rpca_params_default": ([PP, i32], None),
        "rsvd_workspace_bytes": ([vp, MP, PP, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
        "rsvd_run": ([vp, MP, PP, vp, i64, vp, vp, i64], ctypes.c_int),
        "rsvd_run_host": ([vp, MP, PP, vp, i64, vp, vp, i64], ctypes.c_int),
        "rsvd_rqb": ([vp, MP, PP, vp, i64, vp, i64], ctypes.c_int),
        "rsvd_rpca": ([vp, MP, PP, ctypes.POINTER(PcaOut)], ctypes.c_int),
        "rsvd_rpca_host": ([vp, MP, PP, ctypes.POINTER(PcaOut)], ctypes.c_int),
        "rsvd_rpca_predict": ([vp, MP, i32, vp, i64, vp, vp, vp, i64], ctypes.c_int),
        "rsvd_rrpca_params_default": ([ctypes.POINTER(RrpcaParams)], None),
        "rsvd_rid": ([vp, MP, PP, vp, i64, vp, i64, vp], i32),
        "rsvd_rcur": ([vp, MP, PP, vp, i64, vp, i64, vp, i64, vp, vp], i32),
        "rsvd_rrpca": ([vp, MP, ctypes.POINTER(RrpcaParams), vp, vp, i64, ctypes.POINTER(i32),
                        ctypes.POINTER(dp), ctypes.POINTER(dp)], ctypes.c_int),
        "rsvd_rrpca_host": ([vp, MP, ctypes.POINTER(RrpcaParams), vp, vp, i64, ctypes.POINTER(i32),
                             ctypes.POINTER(dp), ctypes.POINTER(dp)], ctypes.c_int),
        "rsvd_omega": ([vp, i64, i64, i32, u64, u64, i32, vp, i64], ctypes.c_int),
        "rsvd_set_profiling": ([vp, ctypes.c_int], ctypes.c_int),
        "rsvd_profile": ([vp, ctypes.c_int, ctypes.POINTER(dp), ctypes.POINTER(i64), ctypes.POINTER(dp)],
                         ctypes.c_int),
        "rsvd_profile_reset": ([vp], ctypes.c_int),
        "rsvd_launch_count": ([vp], i64),
        "rsvd_stats": ([vp, ctypes.POINTER(i64), ctypes.c_int], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


class Context:
    """A library context bound to one CUDA device and stream (default: torch's
    current stream on that device)."""

    def __init__(self, device=None, stream=None):
        L = lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = ctypes.c_void_p()
        st = L.rsvd_create(ctypes.byref(h), self.device.index or 0, ctypes.c_void_p(stream.cuda_stream))
        if st != 0:
            raise RsvdError(st, "rsvd_create failed")
        self.h = h
        self.rank, self.world = 0, 1

    def check(self, st):
        if st != 0:
            raise RsvdError(st, lib().rsvd_last_error(self.h).decode())

    def sync(self):
        """Wait for this context's stream; raise on a numerical failure recorded by
        the calls completed since the last sync (rsvd_sync)."""
        self.check(lib().rsvd_sync(self.h))

    def finish(self, st, sync):
        self.check(st)
        if sync:
            self.sync()

    def last_error(self):
        return lib().rsvd_last_error(self.h).decode()

    def init_group(self, group, rank):
        """Join an in-process RankGroup as `rank` (collectives as fixed-order
        device reductions; one host thread per member context)."""
        self.check(lib().rsvd_comm_init_group(self.h, group.h, int(rank)))
        self.rank, self.world = int(rank), group.n

    def workspace_bytes(self, A, k, p=10, q=2, m_global=None, row_offset=0, center=False, scale=False):
        """Device workspace the library will own for rsvd(A, k, p, q) (rsvd_workspace_bytes)."""
        mat = _matrix(A, m_global, row_offset)
        prm = _params(k, k, k, p, q, "normal", 0, 0, center, scale)
        out = ctypes.c_size_t()
        self.check(lib().rsvd_workspace_bytes(self.h, ctypes.byref(mat), ctypes.byref(prm), ctypes.byref(out)))
        return int(out.value)

    def init_comm(self, rank, world, group=None):
        """NCCL communicator owned by the library: rank 0 makes the unique id,
        torch.distributed broadcasts it (any backend), every rank joins."""
        import torch.distributed as dist
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            self.check(lib().rsvd_nccl_unique_id(buf))
        obj = [bytes(buf.raw)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        raw = ctypes.create_string_buffer(obj[0], 128)
        self.check(lib().rsvd_comm_init(self.h, raw, world, rank))
        self.rank, self.world = rank, world

    def set_profiling(self, on=True):
        """on: False/0 off, True/1 every kind, 2 = the pass kernels only."""
        level = (1 if on else 0) if isinstance(on, bool) else int(on)
        self.check(lib().rsvd_set_profiling(self.h, level))

    def profile(self, kind):
        ms, cnt, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        self.check(lib().rsvd_profile(self.h, kind, ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(by)))
        return ms.value, cnt.value, by.value

    def profile_reset(self):
        self.check(lib().rsvd_profile_reset(self.h))

    def launch_count(self):
        return int(lib().rsvd_launch_count(self.h))

    def stats(self):
        """(Jacobi sweeps, robust re-run taken, kernel launches, Ozaki passes) of the last call."""
        buf = (ctypes.c_int64 * 4)()
        self.check(lib().rsvd_stats(self.h, buf, 4))
        return dict(jacobi_sweeps=int(buf[0]), tsqr_fallback=bool(buf[1]), launches=int(buf[2]),
                    ozaki_passes=int(buf[3]))

    def close(self):
        if getattr(self, "h", None):
            lib().rsvd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RankGroup:
    """In-process rank group (rsvd_group): `n` member contexts, each driven by
    its own host thread, run the row-sharded algorithm together; the
    collectives are fixed-rank-order device reductions."""

    def __init__(self, n):
        h = ctypes.c_void_p()
        st = lib().rsvd_group_create(ctypes.byref(h), int(n))
        if st != 0:
            raise RsvdError(st, "rsvd_group_create(%d) failed" % n)
        self.h, self.n = h, int(n)

    def close(self):
        if getattr(self, "h", None):
            lib().rsvd_group_destroy(self.h)
            self.h = None


def row_partition(m, world):
    """Contiguous row blocks of m rows over `world` ranks: [(offset, rows), ...]."""
    bounds = [(m * r) // world for r in range(world + 1)]
    return [(bounds[r], bounds[r + 1] - bounds[r]) for r in range(world)]


def run_ranks(fn, world, device=None):
    """Run fn(ctx, rank) for rank = 0..world-1 on one device as an in-process
    rank group (one thread and one stream per rank).  Returns the results in
    rank order; re-raises the first exception."""
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    group = RankGroup(world)
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    ctxs = []
    for r in range(world):
        c = Context(dev, streams[r])
        c.init_group(group, r)
        ctxs.append(c)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            with torch.cuda.stream(streams[r]):
                out[r] = fn(ctxs[r], r)
                ctxs[r].sync()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for c in ctxs:
        c.close()
    group.close()
    for e in err:
        if e is not None:
            raise e
    return out


_default_ctx = {}


def default_context(device=None):
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    if key not in _default_ctx:
        _default_ctx[key] = Context(dev, torch.cuda.current_stream(dev))
    return _default_ctx[key]


def _matrix(A, m_global=None, row_offset=0):
    if not A.is_cuda:
        raise ValueError("A must be a CUDA tensor (use the *_host helpers for host buffers)")
    if A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D row-major tensor with unit column stride")
    if A.dtype == torch.float64:
        dt = 0
    elif A.dtype == torch.float32:
        dt = 1
    else:
        raise ValueError("A must be float64 or float32")
    m, n = A.shape
    return Matrix(dt, A.data_ptr(), m, n, A.stride(0), m if m_global is None else m_global, row_offset)


def _params(k, nu, nv, p, q, sdist, seed, stream, center=0, scale=0, power="subspace"):
    prm = Params()
    lib().rsvd_params_default(ctypes.byref(prm), int(k))
    prm.nu = int(k) if nu is None else int(nu)
    prm.nv = int(k) if nv is None else int(nv)
    prm.p, prm.q = int(p), int(q)
    prm.sdist = SDIST[sdist] if isinstance(sdist, str) else int(sdist)
    prm.seed, prm.stream = int(seed), int(stream)
    prm.center, prm.scale = int(bool(center)), int(bool(scale))
    prm.power = POWER[power] if isinstance(power, str) else int(power)
    return prm


RsvdResult = namedtuple("RsvdResult", ["d", "u", "v"])


def rsvd(A, k, nu=None, nv=None, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None,
         m_global=None, row_offset=0, out=None, power="subspace", sync=True):
    """Randomized SVD (Alg. 5; interface P:708).

    power: "subspace" (Alg. 2, QR between passes), "direct" (Alg. 1) or "lu"
    (Alg. 3, pivoted-LU normalisation).
    A: CUDA tensor (m x n, float64 or float32, row-major).  Returns (d, u, v)
    with d (k,), u (m x nu) and v (n x nv, not transposed).  In distributed
    mode (ctx.init_comm) A holds this rank's rows and u this rank's rows.
    """
    ctx = ctx or default_context(A.device)
    mat = _matrix(A, m_global, row_offset)
    mg = mat.m_global
    kk = int(k)
    nu_ = kk if nu is None else min(int(nu), kk)
    nv_ = kk if nv is None else min(int(nv), kk)
    prm = _params(k, nu, nv, p, q, sdist, seed, stream, power=power)
    if out is None:
        d = torch.empty(max(kk, 0), dtype=A.dtype, device=A.device)
        u = torch.empty(A.shape[0], max(nu_, 0), dtype=A.dtype, device=A.device)
        v = torch.empty(A.shape[1], max(nv_, 0), dtype=A.dtype, device=A.device)
    else:
        d, u, v = out
    ctx.finish(lib().rsvd_run(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(u) if nu_ else ctypes.c_void_p(0),
                              max(nu_, 1), _ptr(d), _ptr(v) if nv_ else ctypes.c_void_p(0), max(nv_, 1)), sync)
    return RsvdResult(d, u, v)


def rsvd_host(A_host, k, nu=None, nv=None, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None,
              device="cuda", out=None, m_global=None, row_offset=0):
    """End to end on HOST memory (rsvd_run_host): the library copies A (a CPU
    tensor, pinned for full copy bandwidth) to its device staging buffer,
    factors it and copies (d, u, v) back into CPU tensors (`out` to reuse them)."""
    ctx = ctx or default_context(device)
    if A_host.is_cuda or A_host.dim() != 2 or A_host.stride(1) != 1:
        raise ValueError("A_host must be a 2-D row-major CPU tensor")
    m, n = A_host.shape
    kk = int(k)
    nu_ = kk if nu is None else min(int(nu), kk)
    nv_ = kk if nv is None else min(int(nv), kk)
    dt = 0 if A_host.dtype == torch.float64 else 1
    mat = Matrix(dt, A_host.data_ptr(), m, n, A_host.stride(0), m if m_global is None else m_global, row_offset)
    prm = _params(k, nu_, nv_, p, q, sdist, seed, stream)
    if out is None:
        pin = torch.cuda.is_available()
        d = torch.empty(kk, dtype=A_host.dtype, pin_memory=pin)
        u = torch.empty(m, max(nu_, 0), dtype=A_host.dtype, pin_memory=pin)
        v = torch.empty(n, max(nv_, 0), dtype=A_host.dtype, pin_memory=pin)
    else:
        d, u, v = out
    ctx.check(lib().rsvd_run_host(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(u) if nu_ else ctypes.c_void_p(0),
                                  max(nu_, 1), _ptr(d), _ptr(v) if nv_ else ctypes.c_void_p(0), max(nv_, 1)))
    return RsvdResult(d, u, v)


def rqb(A, k, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None, m_global=None, row_offset=0, sync=True):
    """Randomized QB (Alg. 4): returns (Q (m x l), B (l x n))."""
    ctx = ctx or default_context(A.device)
    mat = _matrix(A, m_global, row_offset)
    l = min(int(k) + int(p), min(mat.m_global, A.shape[1]))
    Q = torch.empty(A.shape[0], l, dtype=A.dtype, device=A.device)
    Bt = torch.empty(A.shape[1], l, dtype=A.dtype, device=A.device)
    prm = _params(k, 0, 0, p, q, sdist, seed, stream)
    ctx.finish(lib().rsvd_rqb(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(Q), l, _ptr(Bt), l), sync)
    return Q, Bt.T


def rid(A, k, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None, m_global=None, row_offset=0, sync=True):
    """Randomized column ID (Alg. rid; Alg. id):
    returns dict(C (m x k) = A[:, J], Z (k x n), J (k,) int64 pivot order)."""
    ctx = ctx or default_context(A.device)
    mat = _matrix(A, m_global, row_offset)
    m, n = A.shape
    kk = int(k)
    C = torch.empty(m, kk, dtype=A.dtype, device=A.device)
    Z = torch.empty(kk, n, dtype=A.dtype, device=A.device)
    J = torch.empty(kk, dtype=torch.int64, device=A.device)
    prm = _params(k, 0, 0, p, q, sdist, seed, stream)
    ctx.finish(lib().rsvd_rid(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(C), kk, _ptr(Z), n, _ptr(J)), sync)
    return dict(C=C, Z=Z, J=J)


def rcur(A, k, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None, sync=True):
    """Randomized CUR (Alg. rcur): A ~ C U R; returns
    dict(C (m x k), U (k x k), R (k x n), J (column indices), I (row indices))."""
    ctx = ctx or default_context(A.device)
    mat = _matrix(A, None, 0)
    m, n = A.shape
    kk = int(k)
    C = torch.empty(m, kk, dtype=A.dtype, device=A.device)
    U = torch.empty(kk, kk, dtype=A.dtype, device=A.device)
    R = torch.empty(kk, n, dtype=A.dtype, device=A.device)
    J = torch.empty(kk, dtype=torch.int64, device=A.device)
    I = torch.empty(kk, dtype=torch.int64, device=A.device)
    prm = _params(k, 0, 0, p, q, sdist, seed, stream)
    ctx.finish(lib().rsvd_rcur(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(C), kk, _ptr(U), kk, _ptr(R), n,
                               _ptr(J), _ptr(I)), sync)
    return dict(C=C, U=U, R=R, J=J, I=I)


def _pca_outputs(m, n, k, dt, dev, retx, center, scale, loadings, whiten, explained, pin=False):
    mk = lambda *shape: torch.empty(*shape, dtype=dt, device=dev, pin_memory=pin)  # noqa: E731
    res = dict(rotation=mk(n, k), eigvals=mk(k), sdev=mk(k), x=mk(m, k) if retx else None,
               center=mk(n) if center else None, scale=mk(n) if scale else None)
    if loadings:
        res["loadings"] = mk(n, k)
    if whiten:
        res["x_white"] = mk(m, k)
    if explained:
        res["var_ratio"], res["var_cum"], res["total_var"] = mk(k), mk(k), mk(1)
    o = PcaOut()
    o.rotation, o.ldr = _ptr(res["rotation"]), k
    o.eigvals, o.sdev = _ptr(res["eigvals"]), _ptr(res["sdev"])
    o.x, o.ldx = _ptr(res["x"]), k
    o.center, o.scale = _ptr(res["center"]), _ptr(res["scale"])
    o.loadings, o.ldl = _ptr(res.get("loadings")), k
    o.x_white, o.ldw = _ptr(res.get("x_white")), k
    o.var_ratio, o.var_cum, o.total_var = _ptr(res.get("var_ratio")), _ptr(res.get("var_cum")), _ptr(res.get("total_var"))
    return res, o


def rpca(A, k, center=True, scale=True, retx=True, p=10, q=2, sdist="normal", seed=0, stream=0, ctx=None,
         m_global=None, row_offset=0, loadings=False, whiten=False, explained=False, sync=True):
    """Randomized PCA (Alg. 6; interface
    rpca(A, k, center=TRUE, scale=TRUE, retx=TRUE, p=10, q=2)).

    Returns dict(rotation, eigvals, sdev, x (retx), center, scale) and, on
    request, loadings = W Lambda^1/2, x_white = the whitened PCs
    (P:1262-1266), var_ratio / var_cum / total_var = the explained variance of
    summary().  Every value is computed by the library.
    A CPU tensor runs end to end through rsvd_rpca_host (outputs on the CPU)."""
    if not A.is_cuda:
        return _rpca_host(A, k, center, scale, retx, p, q, sdist, seed, stream, ctx, loadings, whiten, explained,
                          m_global, row_offset)
    ctx = ctx or default_context(A.device)
    mat = _matrix(A, m_global, row_offset)
    m, n = A.shape
    res, o = _pca_outputs(m, n, int(k), A.dtype, A.device, retx, center, scale, loadings, whiten, explained)
    prm = _params(k, k, k, p, q, sdist, seed, stream, center, scale)
    ctx.finish(lib().rsvd_rpca(ctx.h, ctypes.byref(mat), ctypes.byref(prm), ctypes.byref(o)), sync)
    if explained:
        res["total_var"] = res["total_var"][0]
    return res


def _rpca_host(A, k, center, scale, retx, p, q, sdist, seed, stream, ctx, loadings, whiten, explained,
               m_global=None, row_offset=0):
    ctx = ctx or default_context()
    if A.dim() != 2 or A.stride(1) != 1:
        raise ValueError("A must be a 2-D row-major tensor")
    m, n = A.shape
    dt = 0 if A.dtype == torch.float64 else 1
    mat = Matrix(dt, A.data_ptr(), m, n, A.stride(0), m if m_global is None else m_global, row_offset)
    res, o = _pca_outputs(m, n, int(k), A.dtype, "cpu", retx, center, scale, loadings, whiten, explained,
                          pin=torch.cuda.is_available())
    prm = _params(k, k, k, p, q, sdist, seed, stream, center, scale)
    ctx.check(lib().rsvd_rpca_host(ctx.h, ctypes.byref(mat), ctypes.byref(prm), ctypes.byref(o)))
    if explained:
        res["total_var"] = res["total_var"][0]
    return res


def predict(obj, Anew, ctx=None, sync=True):
    """Out-of-sample projection of an rpca result (predict()):
    ((Anew - center) / scale) @ rotation, by the library's pass kernels."""
    ctx = ctx or default_context(Anew.device)
    mat = _matrix(Anew)
    rot = obj["rotation"]
    kk = rot.shape[1]
    out = torch.empty(Anew.shape[0], kk, dtype=Anew.dtype, device=Anew.device)
    c, s = obj.get("center"), obj.get("scale")
    ctx.finish(lib().rsvd_rpca_predict(ctx.h, ctypes.byref(mat), kk, _ptr(rot), rot.stride(0), _ptr(c), _ptr(s),
                                       _ptr(out), kk), sync)
    return out


def rrpca(A, lam=None, maxiter=50, tol=1e-5, p=10, q=2, k=20, sdist="normal", seed=0, trace=False, ctx=None,
          m_global=None, row_offset=0, rand=True):
    """Randomized robust PCA by inexact ALM (Alg. 7; interface P:1736).

    k > 0 fixes the target rank; k = 0 selects the adaptive target rank of
    Alg. 7 steps (1) and (7) (k = 2, then predict_rank; R30).
    rand=False: the deterministic truncated SVD in step (6).
    trace: per iteration (residual, l, mu, k)."""
    host = not A.is_cuda
    ctx = ctx or default_context(None if host else A.device)
    if host:
        if A.dim() != 2 or not A.is_contiguous():
            raise ValueError("A must be a contiguous 2-D tensor")
        mat = Matrix(0 if A.dtype == torch.float64 else 1, A.data_ptr(), A.shape[0], A.shape[1], A.shape[1],
                     A.shape[0] if m_global is None else m_global, row_offset)
    else:
        mat = _matrix(A, m_global, row_offset)
    prm = RrpcaParams()
    lib().rsvd_rrpca_params_default(ctypes.byref(prm))
    prm.lam = 0.0 if lam is None else float(lam)
    prm.tol, prm.maxiter, prm.k, prm.p, prm.q = float(tol), int(maxiter), int(k), int(p), int(q)
    prm.sdist = SDIST[sdist] if isinstance(sdist, str) else int(sdist)
    prm.seed = int(seed)
    prm.rand = 1 if rand else 0
    pin = host and torch.cuda.is_available()
    L = torch.empty(A.shape, dtype=A.dtype, device=A.device, pin_memory=pin)
    S = torch.empty(A.shape, dtype=A.dtype, device=A.device, pin_memory=pin)
    it = ctypes.c_int32()
    res = ctypes.c_double()
    tr = (ctypes.c_double * (4 * int(maxiter)))()
    fn = lib().rsvd_rrpca_host if host else lib().rsvd_rrpca
    ctx.check(fn(ctx.h, ctypes.byref(mat), ctypes.byref(prm), _ptr(L), _ptr(S), A.shape[1],
                 ctypes.byref(it), ctypes.byref(res), tr))
    hist = [(tr[4 * i], int(tr[4 * i + 1]), tr[4 * i + 2], int(tr[4 * i + 3])) for i in range(it.value)]
    out = dict(L=L, S=S, iters=it.value, residual=res.value)
    if trace:
        out["trace"] = hist
    return out


def omega(n, l, sdist="normal", seed=0, stream=0, dtype=torch.float64, device="cuda", ctx=None):
    """The random test matrix Omega (n x l) from the device generator (K1)."""
    ctx = ctx or default_context(device)
    out = torch.empty(n, l, dtype=dtype, device=device)
    sd = SDIST[sdist] if isinstance(sdist, str) else int(sdist)
    ctx.finish(lib().rsvd_omega(ctx.h, n, l, sd, int(seed), int(stream), 1 if dtype == torch.float32 else 0,
                                _ptr(out), l), True)
    return out


def version():
    return lib().rsvd_version().decode()
