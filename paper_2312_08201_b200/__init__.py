"""B200-native engine for trace(E X(v)) over batches of parameter vectors (arXiv 2312.08201).

    prob = Problem(A0, Bl, Br, Q, E)          # lyap_setup   (offline stage)
    tau = prob.trace_batch(V)                 # lyap_trace_batch (online stage)

A thin ctypes binding over the C-ABI in include/lyapgpu.h (same names; argument marshalling
only — every step runs in the CUDA library liblyapgpu.so).  V may be a NumPy array (host path,
copies inside the call) or a CUDA torch tensor (device path, no copies).  There is no CPU
fallback: without a CUDA device lyap_setup returns LYAP_ENODEV and Problem raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (EXPORTED, LYAP_EPARTIAL, LYAP_KMAX, LYAP_OK, Info, LyapError, Opts, Stats, lib)

__all__ = ["Problem", "EKProblem", "LyapError", "lib", "EXPORTED", "LYAP_KMAX", "default_opts"]


def default_opts() -> Opts:
    o = Opts()
    lib.lyap_default_opts(C.byref(o))
    return o


def _f64(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Problem:
    """One seed A0 with its factors (lyap_setup); trace_batch evaluates trace(E X(v)).  Q may be (n, n),
    or (k, n, n) for a right-hand side linear in v, Q(v) = sum_i v_i Q[i] (lyap_setup_qlin)."""

    def __init__(self, A0, Bl, Br, Q, E, *, tol: float = 1e-12, max_dim: int = 0, max_restarts: int = 30,
                 batch: int = 0, warm_start: bool = False, max_cond_S: float = 1e8, device: int = -1,
                 profile: bool = False, schedule: bool = True, recycle: int = -1, check_stable: bool = False,
                 coarse: int = -1, mixed: int = -1, mixed_eta: float = 1e-4):
        A0 = _f64(A0)
        n = A0.shape[0]
        Bl = _f64(Bl)
        if Bl.ndim == 1:
            Bl = Bl[:, None]
        k = Bl.shape[1]
        Br = _f64(Br).reshape(n, k)
        Bl = Bl.reshape(n, k)
        E = _f64(E, (n, n))
        Q = _f64(Q)
        qlin = Q.ndim == 3  # (k, n, n): Q(v) = sum_i v_i Q[i]  (lyap_setup_qlin)
        if qlin and Q.shape != (k, n, n):
            raise ValueError(f"a v-linear Q must be ({k}, {n}, {n})")
        if not qlin:
            Q = _f64(Q, (n, n))
        o = default_opts()
        o.tol, o.max_dim, o.max_restarts, o.batch = tol, max_dim, max_restarts, batch
        o.warm_start, o.max_cond_S, o.device, o.profile = int(warm_start), max_cond_S, device, int(profile)
        o.schedule = int(schedule)
        o.recycle = int(recycle)
        o.check_stable = int(check_stable)
        o.coarse = int(coarse)
        o.mixed, o.mixed_eta = int(mixed), float(mixed_eta)
        self._ctx = C.c_void_p()
        setup = lib.lyap_setup_qlin if qlin else lib.lyap_setup
        rc = setup(n, k, _dp(A0), _dp(Bl), _dp(Br), _dp(Q), _dp(E), C.byref(o), C.byref(self._ctx))
        if rc != LYAP_OK:
            raise LyapError(rc, lib.lyap_last_error(None).decode())
        self.n, self.k = n, k
        # mixed-precision mode in effect (opts.mixed -1 = auto: on for n > 1536)
        self.mixed = int(mixed) if int(mixed) >= 0 else int(n > 1536)

    def like(self, Bl, Br=None) -> "Problem":
        """Same A0, Q, E with another (Bl, Br) configuration (NEXT row f4): reuses this problem's
        eigendecomposition and seed basis (lyap_setup_like)."""
        Bl = _f64(Bl)
        if Bl.ndim == 1:
            Bl = Bl[:, None]
        Br = Bl if Br is None else _f64(Br).reshape(Bl.shape)
        new = Problem.__new__(Problem)
        new._ctx = C.c_void_p()
        rc = lib.lyap_setup_like(self._ctx, Bl.shape[1], _dp(Bl), _dp(Br), None, C.byref(new._ctx))
        if rc != LYAP_OK:
            raise LyapError(rc, lib.lyap_last_error(None).decode())
        new.n, new.k = self.n, Bl.shape[1]
        return new

    # ------------------------------------------------------------------ queries
    @property
    def info(self) -> dict:
        i = Info()
        self._check(lib.lyap_get_info(self._ctx, C.byref(i)))
        d = {f: getattr(i, f) for f, _ in Info._fields_}
        d["wcost"] = list(d["wcost"])[: d["k"]]
        return d

    def cost_proxy(self, V) -> np.ndarray:
        """The engine's per-v cost proxy sum_t |v_t| ||B~l_t|| ||B^r_t|| (the scheduling key of
        lyap_trace_batch; used to balance multi-GPU shards)."""
        V = np.asarray(V, dtype=np.float64).reshape(-1, self.k)
        return np.abs(V) @ np.asarray(self.info["wcost"])

    @property
    def stats(self) -> dict:
        s = Stats()
        self._check(lib.lyap_get_stats(self._ctx, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def reset_stats(self):
        self._check(lib.lyap_reset_stats(self._ctx))

    def _check(self, rc):
        if rc != LYAP_OK:
            raise LyapError(rc, lib.lyap_last_error(self._ctx).decode())

    # ------------------------------------------------------------------ online stage
    def trace_batch(self, V, *, return_diagnostics: bool = False, allow_partial: bool = False, stream=None):
        """tau[i] = trace(E X(V[i])).  V: (nv, k) NumPy array (host path) or CUDA torch tensor.

        With return_diagnostics: (tau, status, applies, resid).  A non-zero status raises
        LyapError(LYAP_EPARTIAL) unless allow_partial."""
        try:
            import torch
            is_dev = isinstance(V, torch.Tensor) and V.is_cuda
        except ImportError:  # pragma: no cover
            is_dev = False
        if is_dev:
            return self._trace_batch_device(V, return_diagnostics, allow_partial, stream)
        V = _f64(V)
        if V.ndim == 1:
            V = V.reshape(-1, self.k)
        nv = V.shape[0]
        if V.shape[1] != self.k:
            raise ValueError(f"V must be (nv, {self.k})")
        tau = np.empty(nv)
        st = np.empty(nv, dtype=np.int32)
        ap = np.empty(nv, dtype=np.int32)
        rs = np.empty(nv)
        rc = lib.lyap_trace_batch_ex(self._ctx, nv, V.ctypes.data, tau.ctypes.data, st.ctypes.data,
                                     ap.ctypes.data, rs.ctypes.data, 0, None)
        if rc != LYAP_OK and not (rc == LYAP_EPARTIAL and allow_partial):
            self._check(rc)
        return (tau, st, ap, rs) if return_diagnostics else tau

    def _trace_batch_device(self, V, return_diagnostics, allow_partial, stream):
        import torch
        V = V.to(torch.float64)
        if V.ndim == 1:
            V = V.reshape(-1, self.k)
        if V.ndim != 2 or V.shape[1] != self.k:
            raise ValueError(f"V must be (nv, {self.k}), got {tuple(V.shape)}")
        V = V.contiguous()
        nv = V.shape[0]
        dev = V.device
        tau = torch.empty(nv, dtype=torch.float64, device=dev)
        st = torch.empty(nv, dtype=torch.int32, device=dev)
        ap = torch.empty(nv, dtype=torch.int32, device=dev)
        rs = torch.empty(nv, dtype=torch.float64, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        rc = lib.lyap_trace_batch_ex(self._ctx, nv, V.data_ptr(), tau.data_ptr(), st.data_ptr(), ap.data_ptr(),
                                     rs.data_ptr(), 1, C.c_void_p(s.cuda_stream))
        if rc != LYAP_OK and not (rc == LYAP_EPARTIAL and allow_partial):
            self._check(rc)
        return (tau, st, ap, rs) if return_diagnostics else tau

    def trace_batch_x(self, V, x0=None, *, return_diagnostics: bool = False, allow_partial: bool = False,
                      stream=None):
        """Device path with solution recycling (lyap_trace_batch_x, NEXT row f3): V (nv, k) CUDA tensor,
        x0 (nv, k, npad) CUDA tensor of initial guesses or None.  Returns (tau, G) with G (nv, k, npad)
        the folded solutions (pass them back as x0 for nearby v); with return_diagnostics also
        (status, applies, resid)."""
        import torch
        V = V.to(torch.float64)
        if V.ndim == 1:
            V = V.reshape(-1, self.k)
        if V.ndim != 2 or V.shape[1] != self.k:
            raise ValueError(f"V must be (nv, {self.k}), got {tuple(V.shape)}")
        V = V.contiguous()
        nv, dev = V.shape[0], V.device
        npad = self.info["npad"]
        if x0 is not None:
            x0 = x0.to(torch.float64).contiguous()
            if tuple(x0.shape) != (nv, self.k, npad):
                raise ValueError(f"x0 must be ({nv}, {self.k}, {npad})")
        tau = torch.empty(nv, dtype=torch.float64, device=dev)
        G = torch.zeros(nv, self.k, npad, dtype=torch.float64, device=dev)
        st = torch.empty(nv, dtype=torch.int32, device=dev)
        ap = torch.empty(nv, dtype=torch.int32, device=dev)
        rs = torch.empty(nv, dtype=torch.float64, device=dev)
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        rc = lib.lyap_trace_batch_x(self._ctx, nv, V.data_ptr(), x0.data_ptr() if x0 is not None else None,
                                    G.data_ptr(), tau.data_ptr(), st.data_ptr(), ap.data_ptr(), rs.data_ptr(),
                                    C.c_void_p(s.cuda_stream))
        if rc != LYAP_OK and not (rc == LYAP_EPARTIAL and allow_partial):
            self._check(rc)
        return (tau, G, st, ap, rs) if return_diagnostics else (tau, G)

    def unstable_count(self, V) -> np.ndarray:
        """NEXT row f4 (lyap_stable_batch): per row of V the number of eigenvalues of A(v) in the open
        right half-plane (-1: on / numerically at the imaginary axis).  Stable iff 0."""
        V = _f64(V)
        if V.ndim == 1:
            V = V.reshape(-1, self.k)
        out = np.empty(V.shape[0], dtype=np.int32)
        self._check(lib.lyap_stable_batch(self._ctx, V.shape[0], V.ctypes.data, out.ctypes.data, 0, None))
        return out

    def solution(self, V, return_traces: bool = False):
        """Full X(v) (n x n) for each row of V (NEXT row f2; O(n^3) per v).  Returns (nv, n, n)."""
        V = _f64(V)
        if V.ndim == 1:
            V = V.reshape(-1, self.k)
        nv = V.shape[0]
        X = np.empty((nv, self.n, self.n))
        tau = np.empty(nv)
        self._check(lib.lyap_solution(self._ctx, nv, V.ctypes.data, X.ctypes.data, tau.ctypes.data))
        return (X, tau) if return_traces else X

    def build_recycle(self, seeds=None, V=None, s: int = 32):
        """Recycle spaces from one recorded GMRES cycle per seed (lyap_build_recycle).  seeds (nseeds, k);
        or V: use the 2^k corners of the bounding box of the rows of V (positive parameters)."""
        if seeds is None:
            V = _f64(V).reshape(-1, self.k)
            lo, hi = V.min(axis=0), V.max(axis=0)
            import itertools
            seeds = np.array([[hi[t] if b else lo[t] for t, b in enumerate(bits)]
                              for bits in itertools.product((0, 1), repeat=self.k)])
        seeds = _f64(seeds).reshape(-1, self.k)
        self._check(lib.lyap_build_recycle(self._ctx, seeds.shape[0], seeds.ctypes.data, s))

    def set_recycle(self, U, seeds):
        """Recycle spaces: U (nreg, s, k, npad) folded x-space vectors, seeds (nreg, k)."""
        U = _f64(U)
        seeds = _f64(seeds).reshape(U.shape[0], self.k)
        self._check(lib.lyap_set_recycle(self._ctx, U.shape[0], U.shape[1], U.ctypes.data, seeds.ctypes.data))

    def apply_C(self, X, sigma=None, stream=None, mixed=False):
        """K1 alone: Y = sigma o X - T X for folded vectors X (CUDA tensor, (nvec, k, npad)).
        mixed=True: the 3xTF32 tcgen05 operator of the mixed-precision Krylov steps (lyap_apply_C_mixed)."""
        import torch
        X = X.to(torch.float64).contiguous()
        Y = torch.empty_like(X)
        sp = None
        if sigma is not None:
            sigma = sigma.to(torch.float64).contiguous()
            sp = sigma.data_ptr()
        s = stream if stream is not None else torch.cuda.current_stream(X.device)
        fn = lib.lyap_apply_C_mixed if mixed else lib.lyap_apply_C
        self._check(fn(self._ctx, X.shape[0], X.data_ptr(), sp, Y.data_ptr(), C.c_void_p(s.cuda_stream)))
        return Y

    def export_state(self) -> dict:
        i = self.info
        n, k, npad, npairs = i["n"], i["k"], i["npad"], i["n_pairs"]
        nrep = n - npairs
        out = {"lam": np.empty((n, 2)), "bhr": np.empty((n, k)), "btl": np.empty((n, k)),
               "F": np.empty((nrep, k, k, 2)), "g0": np.empty((k, npad)), "hf": np.empty((k, npad))}
        self._check(lib.lyap_export_state(self._ctx, *(out[x].ctypes.data for x in
                                                       ("lam", "bhr", "btl", "F", "g0", "hf"))))
        out.update(t0=i["t0"], n_pairs=npairs, npad=npad)
        return out

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            lib.lyap_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class EKProblem:
    """NEXT row f1: extended-Krylov projection (§2.2, Alg. 1) for large n.  X0Br = X0 @ Br of
    the seed solution, trEX0 = trace(E X0).  trace_batch(V, eps) -> approximate traces."""

    def __init__(self, A0, Bl, Br, X0Br, E, trEX0: float, max_dim: int = 0):
        A0 = _f64(A0)
        n = A0.shape[0]
        Bl = _f64(Bl).reshape(n, -1)
        k = Bl.shape[1]
        Br, X0Br, E = _f64(Br).reshape(n, k), _f64(X0Br).reshape(n, k), _f64(E, (n, n))
        self._ek = C.c_void_p()
        rc = lib.lyap_ek_setup(n, k, _dp(A0), _dp(Bl), _dp(Br), _dp(X0Br), _dp(E), float(trEX0), max_dim,
                               C.byref(self._ek))
        if rc != LYAP_OK:
            raise LyapError(rc, lib.lyap_ek_last_error(None).decode())
        self.n, self.k = n, k

    def trace_batch(self, V, eps: float = 1e-8, max_steps: int = 200, allow_partial: bool = False,
                    per_v: bool = False):
        """(traces, basis dim, certified backward error).  LYAP_EPARTIAL (target not certified) raises
        unless allow_partial.  per_v: (traces, backward error per v, basis size per v) -- Alg. 1's
        per-v certification (lyap_ek_trace_batch_ex)."""
        V = _f64(V).reshape(-1, self.k)
        if per_v:
            tau = np.empty(V.shape[0])
            bw = np.empty(V.shape[0])
            dm = np.empty(V.shape[0], dtype=np.int32)
            rc = lib.lyap_ek_trace_batch_ex(self._ek, V.shape[0], V.ctypes.data, eps, max_steps, tau.ctypes.data,
                                            bw.ctypes.data, dm.ctypes.data)
            if rc != LYAP_OK and not (rc == LYAP_EPARTIAL and allow_partial):
                raise LyapError(rc, lib.lyap_ek_last_error(self._ek).decode())
            return tau, bw, dm
        tau = np.empty(V.shape[0])
        dim = C.c_int32()
        err = C.c_double()
        rc = lib.lyap_ek_trace_batch(self._ek, V.shape[0], V.ctypes.data, eps, max_steps, tau.ctypes.data,
                                     C.byref(dim), C.byref(err))
        if rc != LYAP_OK and not (rc == LYAP_EPARTIAL and allow_partial):
            raise LyapError(rc, lib.lyap_ek_last_error(self._ek).decode())
        return tau, int(dim.value), float(err.value)

    def close(self):
        if getattr(self, "_ek", None) and self._ek.value:
            lib.lyap_ek_destroy(self._ek)
            self._ek = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
