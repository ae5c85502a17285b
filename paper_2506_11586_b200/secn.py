"""Thin Python binding of libsecn (include/secn.h): argument marshalling only.

Every step of the hot path runs in libsecn's CUDA kernels; this module only checks tensor
shapes/dtypes, passes device pointers and the current torch CUDA stream through ctypes,
and raises on a non-OK status. Tensors hold the uint64 residues in int64 storage (PyTorch's
uint64 support is partial); values are never interpreted here. There is no CPU fallback:
if libsecn.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import build as _build

# Reading R1: N = 4096, q0 = 2^60 - 2^14 + 1, q1 = 2^49 - 204799, t = 2^37.
DEFAULT_LOG_N = 12
DEFAULT_PRIMES = (0x0FFFFFFFFFFFC001, 0x1FFFFFFFCE001)
DEFAULT_T_BITS = 37
# Reading R1b: 32-bit RNS limbs -- the four largest 27-bit primes = 1 mod 2^16.
DEFAULT_PRIMES32 = (0x7E90001, 0x7E00001, 0x7DD0001, 0x7D70001)

SECN_MAX_LIMBS = 4
STATUS = {0: "SECN_OK", -1: "SECN_EINVAL", -2: "SECN_EUNSUPPORTED", -3: "SECN_ERANGE", -4: "SECN_ENOMEM",
          -5: "SECN_ECUDA", -6: "SECN_ESTATE"}

EXPORTS = ("secn_ctx_create", "secn_ctx_destroy", "secn_ctx_query", "secn_last_error", "secn_conv_plan",
           "secn_conv_plan_ex",
           "secn_ntt_fwd", "secn_ntt_inv", "secn_preprocess_weights", "secn_share_add", "secn_mask_add",
           "secn_he_conv2d_workspace", "secn_he_conv2d", "secn_he_conv2d_stage", "secn_extract_share",
           "secn32_ctx_create", "secn32_ntt_fwd", "secn32_ntt_inv", "secn32_preprocess_weights",
           "secn32_share_add", "secn32_mask_add", "secn32_he_conv2d", "secn32_he_conv2d_stage",
           "secn_he_conv2d_stage_ex", "secn32_he_conv2d_stage_ex",
           "secn_he_conv2d_ex", "secn32_he_conv2d_ex", "secn_he_conv2d_online_workspace",
           "secn_he_conv2d_online", "secn32_he_conv2d_online", "secn_fc_plan", "secn_fc_preprocess_weights",
           "secn32_fc_preprocess_weights", "secn_he_fc_workspace", "secn_he_fc", "secn32_he_fc",
           "secn_he_conv2d_lwe_workspace", "secn_he_conv2d_lwe", "secn32_he_conv2d_lwe", "secn_he_fc_lwe_workspace",
           "secn_he_fc_lwe", "secn32_he_fc_lwe", "secn_mask_draw", "secn_he_conv2d_gen_workspace", "secn_he_conv2d_gen",
           "secn32_he_conv2d_gen", "secn_he_conv2d_lwe_gen_workspace", "secn_he_conv2d_lwe_gen", "secn32_he_conv2d_lwe_gen",
           "secn_mask_encoded_bytes", "secn_mask_encode", "secn_he_conv2d_em", "secn32_he_conv2d_em",
           "secn_he_conv2d_lwe_em", "secn32_he_conv2d_lwe_em")


class SecnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class FcPlan(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in ("n_i", "n_o", "nib", "nob", "G", "M")]

    def __repr__(self):
        return "FcPlan(" + ", ".join(f"{f}={getattr(self, f)}" for f, _ in self._fields_) + ")"


class MaskGen(ctypes.Structure):
    """secn_mask_gen_t (reading R17): Philox4x32-10 key `seed`, stream id, first output ct index."""
    _fields_ = [("seed", ctypes.c_uint64), ("stream", ctypes.c_uint32), ("ct0", ctypes.c_uint32)]


class Plan(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint32) for f in
                ("C", "H", "W", "M", "kh", "kw", "stride", "pad", "Hw", "Ww", "OH", "OW", "decim", "Hp", "Wp",
                 "Cw", "G", "S", "nbh", "nbw", "O", "s_begin", "s_count")]

    def copy(self, **kw) -> "Plan":
        p = Plan()
        ctypes.pointer(p)[0] = self
        for k, v in kw.items():
            setattr(p, k, v)
        return p

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}

    def __repr__(self):
        return "Plan(" + ", ".join(f"{k}={v}" for k, v in self.as_dict().items()) + ")"


class CtxInfo(ctypes.Structure):
    _fields_ = [("log_n", ctypes.c_uint32), ("n", ctypes.c_uint32), ("n_limbs", ctypes.c_uint32),
                ("t_bits", ctypes.c_uint32), ("primes", ctypes.c_uint64 * SECN_MAX_LIMBS),
                ("psi", ctypes.c_uint64 * SECN_MAX_LIMBS), ("device", ctypes.c_int), ("word_bits", ctypes.c_uint32)]


_lib = None


def lib(path=None) -> ctypes.CDLL:
    """Loads libsecn.so (built by __graft_entry__.build()); raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or _build.LIB
    if not p.exists():
        raise RuntimeError(f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(str(p))
    vp, i, u32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_size_t
    P = ctypes.POINTER(Plan)
    sig = {
        "secn_ctx_create": (i, [ctypes.POINTER(vp), i, u32, u32, ctypes.POINTER(ctypes.c_uint64), u32]),
        "secn_ctx_destroy": (i, [vp]),
        "secn_ctx_query": (i, [vp, ctypes.POINTER(CtxInfo)]),
        "secn_last_error": (ctypes.c_char_p, []),
        "secn_conv_plan": (i, [u32, u32, P]),
        "secn_conv_plan_ex": (i, [u32, u32, u32, P]),
        "secn_ntt_fwd": (i, [vp, vp, sz, vp]),
        "secn_ntt_inv": (i, [vp, vp, sz, vp]),
        "secn_preprocess_weights": (i, [vp, P, vp, vp, vp]),
        "secn_share_add": (i, [vp, vp, vp, sz, vp]),
        "secn_mask_add": (i, [vp, vp, vp, sz, vp]),
        "secn_he_conv2d_workspace": (sz, [vp, P]),
        "secn_he_conv2d": (i, [vp, P, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_stage": (i, [vp, P, i, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_stage_ex": (i, [vp, P, i, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_ex": (i, [vp, P, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_online_workspace": (sz, [vp, P]),
        "secn_fc_plan": (i, [u32, u32, ctypes.POINTER(FcPlan)]),
        "secn_he_conv2d_lwe_workspace": (sz, [vp, P]),
        "secn_he_conv2d_lwe": (i, [vp, P, vp, vp, vp, vp, u32, vp, vp, vp, vp, sz, vp]),
        "secn_he_fc_lwe_workspace": (sz, [vp, ctypes.POINTER(FcPlan)]),
        "secn_he_fc_lwe": (i, [vp, ctypes.POINTER(FcPlan), vp, vp, vp, vp, u32, vp, vp, vp, vp, sz, vp]),
        "secn_fc_preprocess_weights": (i, [vp, ctypes.POINTER(FcPlan), vp, vp, vp]),
        "secn_he_fc_workspace": (sz, [vp, ctypes.POINTER(FcPlan)]),
        "secn_he_fc": (i, [vp, ctypes.POINTER(FcPlan), vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_online": (i, [vp, P, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_extract_share": (i, [vp, P, vp, vp, vp]),
        "secn32_ctx_create": (i, [ctypes.POINTER(vp), i, u32, u32, ctypes.POINTER(ctypes.c_uint32), u32]),
        "secn_mask_draw": (i, [vp, ctypes.POINTER(MaskGen), sz, vp, vp]),
        "secn_he_conv2d_gen_workspace": (sz, [vp, P]),
        "secn_he_conv2d_gen": (i, [vp, P, vp, vp, vp, ctypes.POINTER(MaskGen), vp, vp, vp, sz, vp]),
        "secn_he_conv2d_lwe_gen_workspace": (sz, [vp, P]),
        "secn_he_conv2d_lwe_gen": (i, [vp, P, vp, vp, vp, ctypes.POINTER(MaskGen), u32, vp, vp, vp, vp, sz, vp]),
        "secn_mask_encoded_bytes": (sz, [vp, P]),
        "secn_mask_encode": (i, [vp, P, vp, ctypes.POINTER(MaskGen), vp, vp, vp]),
        "secn_he_conv2d_em": (i, [vp, P, vp, vp, vp, vp, vp, vp, sz, vp]),
        "secn_he_conv2d_lwe_em": (i, [vp, P, vp, vp, vp, vp, u32, vp, vp, vp, sz, vp]),
    }
    for f in ("ntt_fwd", "ntt_inv", "preprocess_weights", "share_add", "mask_add", "he_conv2d", "he_conv2d_stage",
              "he_conv2d_stage_ex", "he_conv2d_ex",
              "he_conv2d_online", "fc_preprocess_weights", "he_fc", "he_conv2d_lwe", "he_fc_lwe", "he_conv2d_gen",
              "he_conv2d_lwe_gen", "he_conv2d_em", "he_conv2d_lwe_em"):
        sig["secn32_" + f] = sig["secn_" + f]
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    if path is None:
        _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise SecnError(status, lib().secn_last_error().decode())


PLAN_BYTES, PLAN_TIME = 0, 1  # SECN_PLAN_BYTES (reading R6), SECN_PLAN_TIME (reading R6b)


def conv_plan(C, H, W, M, kh, kw=None, stride=1, pad=0, log_n=DEFAULT_LOG_N, n_limbs=len(DEFAULT_PRIMES),
              Hw=0, Ww=0, rule=PLAN_TIME) -> Plan:
    """secn_conv_plan_ex: packing plan of one conv layer (rule PLAN_TIME: modelled device time,
    reading R6b, the default; PLAN_BYTES: byte-min, reading R6; explicit Hw, Ww are validated)."""
    p = Plan(C=C, H=H, W=W, M=M, kh=kh, kw=kh if kw is None else kw, stride=stride, pad=pad, Hw=Hw, Ww=Ww)
    _check(lib().secn_conv_plan_ex(log_n, n_limbs, rule, ctypes.byref(p)))
    return p


def fc_plan(n_i, n_o, log_n=DEFAULT_LOG_N, coef_words64=len(DEFAULT_PRIMES), nib=0) -> FcPlan:
    """secn_fc_plan: matrix-vector packing of an n_o x n_i fully-connected layer (reading R15)."""
    p = FcPlan(n_i=n_i, n_o=n_o, nib=nib)
    _check(lib().secn_fc_plan(log_n, coef_words64, ctypes.byref(p)))
    return p


def _ptr(t: Optional[torch.Tensor], shape=None, name="tensor", dtype=torch.int64):
    if t is None:
        return None
    if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous {dtype} CUDA tensor, got {t.dtype} {t.device}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


def _ws(t: torch.Tensor, need: int, device) -> tuple:
    """(pointer, bytes) of a caller's workspace tensor after checking it is a contiguous CUDA tensor
    on the context's device with at least `need` bytes (the C ABI cannot see its size)."""
    if not t.is_cuda or not t.is_contiguous() or t.device != device:
        raise TypeError(f"workspace: expected a contiguous CUDA tensor on {device}, got {t.device}")
    nb = t.numel() * t.element_size()
    if nb < need:
        raise ValueError(f"workspace: {nb} bytes < the {need} the call needs")
    return ctypes.c_void_p(t.data_ptr()), nb


class Context:
    """A libsecn context on one CUDA device (secn_ctx_create, or secn32_ctx_create with
    word_bits=32). Residue tensors are int64 (64-bit words) or int32 (32-bit words); plaintext
    side tensors (x0, r, kernels, y0) are always int64."""

    def __init__(self, device: int = 0, log_n: int = DEFAULT_LOG_N, primes: Optional[Sequence[int]] = None,
                 t_bits: int = DEFAULT_T_BITS, word_bits: int = 64):
        if word_bits not in (32, 64):
            raise ValueError("word_bits must be 32 or 64")
        if primes is None:
            primes = DEFAULT_PRIMES if word_bits == 64 else DEFAULT_PRIMES32
        self._h = ctypes.c_void_p()
        self.word_bits = word_bits
        self.rdtype = torch.int64 if word_bits == 64 else torch.int32
        self._pre = "secn_" if word_bits == 64 else "secn32_"
        if word_bits == 64:
            arr = (ctypes.c_uint64 * len(primes))(*primes)
            _check(lib().secn_ctx_create(ctypes.byref(self._h), device, log_n, len(primes), arr, t_bits))
        else:
            arr = (ctypes.c_uint32 * len(primes))(*primes)
            _check(lib().secn32_ctx_create(ctypes.byref(self._h), device, log_n, len(primes), arr, t_bits))
        info = CtxInfo()
        _check(lib().secn_ctx_query(self._h, ctypes.byref(info)))
        self.device = torch.device("cuda", device)
        self.log_n, self.n, self.L, self.t_bits = info.log_n, info.n, info.n_limbs, info.t_bits
        self.primes = tuple(info.primes[: self.L])
        self.psi = tuple(info.psi[: self.L])

    def _f(self, name):
        return getattr(lib(), self._pre + name)

    def _rp(self, t, shape=None, name="residues"):
        return _ptr(t, shape, name, self.rdtype)

    def empty(self, *shape) -> torch.Tensor:
        """An uninitialised residue tensor of this context's word size."""
        return torch.empty(shape, dtype=self.rdtype, device=self.device)

    def close(self):
        if self._h:
            lib().secn_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self, stream):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    @property
    def coef_words64(self) -> int:
        """8-byte words per coefficient of a ciphertext component (the plan's byte model)."""
        return max(1, self.L * self.word_bits // 64)

    def plan(self, C, H, W, M, kh, kw=None, stride=1, pad=0, Hw=0, Ww=0, rule=PLAN_TIME) -> Plan:
        return conv_plan(C, H, W, M, kh, kw, stride, pad, self.log_n, self.coef_words64, Hw, Ww, rule)

    # -- boundary calls ---------------------------------------------------------------------
    def ntt_fwd(self, polys: torch.Tensor, stream=None) -> torch.Tensor:
        n = polys.numel() // (self.L * self.n)
        _check(self._f("ntt_fwd")(self._h, self._rp(polys, None, "polys"), n, self._stream(stream)))
        return polys

    def ntt_inv(self, polys: torch.Tensor, stream=None) -> torch.Tensor:
        n = polys.numel() // (self.L * self.n)
        _check(self._f("ntt_inv")(self._h, self._rp(polys, None, "polys"), n, self._stream(stream)))
        return polys

    def preprocess_weights(self, plan: Plan, kernel: torch.Tensor, out: Optional[torch.Tensor] = None,
                           stream=None) -> torch.Tensor:
        shape = (plan.M, plan.G, self.L, self.n)
        if out is None:
            out = self.empty(*shape)
        _check(self._f("preprocess_weights")(self._h, ctypes.byref(plan),
                                             _ptr(kernel, (plan.M, plan.C, plan.kh, plan.kw), "kernel"),
                                             self._rp(out, shape, "w_ntt"), self._stream(stream)))
        return out

    # ---- fully connected (f3) ----
    def fc_plan(self, n_i: int, n_o: int, nib: int = 0) -> FcPlan:
        return fc_plan(n_i, n_o, self.log_n, self.coef_words64, nib)

    def fc_preprocess_weights(self, plan: FcPlan, W: torch.Tensor, out: Optional[torch.Tensor] = None,
                              stream=None) -> torch.Tensor:
        """W int64 [n_o][n_i] (< 2^t) -> w_ntt [M][G][L][N] (NTT domain)."""
        shape = (plan.M, plan.G, self.L, self.n)
        if out is None:
            out = self.empty(*shape)
        _check(self._f("fc_preprocess_weights")(self._h, ctypes.byref(plan), _ptr(W, (plan.n_o, plan.n_i), "W"),
                                                self._rp(out, shape, "w_ntt"), self._stream(stream)))
        return out

    def he_fc(self, plan: FcPlan, ct_in: torch.Tensor, w_ntt: torch.Tensor, x0: Optional[torch.Tensor] = None,
              r: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
              y0: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
              stream=None) -> torch.Tensor:
        """secn_he_fc: ct_in [G][2][L][N] -> ct_out [M][2][L][N]; y0 int64 [n_o] (server share)."""
        L, n = self.L, self.n
        if out is None:
            out = self.empty(plan.M, 2, L, n)
        need = int(lib().secn_he_fc_workspace(self._h, ctypes.byref(plan)))
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_fc")(self._h, ctypes.byref(plan), self._rp(ct_in, (plan.G, 2, L, n), "ct_in"),
                                _ptr(x0, (plan.G, n), "x0"), self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"),
                                _ptr(r, (plan.M, n), "r"), self._rp(out, (plan.M, 2, L, n), "ct_out"),
                                _ptr(y0, (plan.n_o,), "y0"), wp, wn, self._stream(stream)))
        return out

    # ---- extracted outputs (f2): modulus switch to `keep` limbs + designated coefficients ----
    def he_conv2d_lwe(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, keep: int,
                      x0: Optional[torch.Tensor] = None, r: Optional[torch.Tensor] = None,
                      y0: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None, stream=None,
                      out: Optional[tuple] = None):
        """secn_he_conv2d_lwe -> (a' [M*S][keep][N], b' [M][OH][OW][keep]) in the residue dtype
        (written into `out` = (a', b') when given)."""
        L, n = self.L, self.n
        a, b = out if out is not None else (self.empty(plan.M * plan.S, keep, n), self.empty(plan.M, plan.OH, plan.OW, keep))
        need = int(lib().secn_he_conv2d_lwe_workspace(self._h, ctypes.byref(plan)))
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_lwe")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (plan.G * plan.S, 2, L, n), "ct_in"),
            _ptr(x0, (plan.G * plan.S, n), "x0"), self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"),
            _ptr(r, (plan.M * plan.S, n), "r"), keep, self._rp(a, (plan.M * plan.S, keep, n), "a_out"),
            self._rp(b, (plan.M, plan.OH, plan.OW, keep), "b_out"),
            _ptr(y0, (plan.M, plan.OH, plan.OW), "y0"), wp, wn, self._stream(stream)))
        return a, b

    def he_fc_lwe(self, plan: FcPlan, ct_in: torch.Tensor, w_ntt: torch.Tensor, keep: int,
                  x0: Optional[torch.Tensor] = None, r: Optional[torch.Tensor] = None,
                  y0: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None, stream=None):
        """secn_he_fc_lwe -> (a' [M][keep][N], b' [n_o][keep])."""
        L, n = self.L, self.n
        a = self.empty(plan.M, keep, n)
        b = self.empty(plan.n_o, keep)
        need = int(lib().secn_he_fc_lwe_workspace(self._h, ctypes.byref(plan)))
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_fc_lwe")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (plan.G, 2, L, n), "ct_in"), _ptr(x0, (plan.G, n), "x0"),
            self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), _ptr(r, (plan.M, n), "r"), keep,
            self._rp(a, (plan.M, keep, n), "a_out"), self._rp(b, (plan.n_o, keep), "b_out"),
            _ptr(y0, (plan.n_o,), "y0"), wp, wn, self._stream(stream)))
        return a, b

    def share_add(self, ct: torch.Tensor, x0: torch.Tensor, stream=None) -> torch.Tensor:
        n = ct.shape[0]
        _check(self._f("share_add")(self._h, self._rp(ct, (n, 2, self.L, self.n), "ct"), _ptr(x0, (n, self.n), "x0"),
                                    n, self._stream(stream)))
        return ct

    def mask_add(self, ct: torch.Tensor, r: torch.Tensor, stream=None) -> torch.Tensor:
        n = ct.shape[0]
        _check(self._f("mask_add")(self._h, self._rp(ct, (n, 2, self.L, self.n), "ct"), _ptr(r, (n, self.n), "r"), n,
                                   self._stream(stream)))
        return ct

    def workspace_bytes(self, plan: Plan) -> int:
        return lib().secn_he_conv2d_workspace(self._h, ctypes.byref(plan))

    def he_conv2d(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, x0: Optional[torch.Tensor] = None,
                  r: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None, stream=None, y0: Optional[torch.Tensor] = None
                  ) -> torch.Tensor:
        """secn_he_conv2d; with y0 (int64 [M][OH][OW]) secn_he_conv2d_ex, which also writes the
        server's output share in the same launches."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        if out is None:
            out = self.empty(n_out, 2, L, n)
        ws_bytes = self.workspace_bytes(plan)
        if workspace is None:
            workspace = torch.empty((ws_bytes + 7) // 8, dtype=torch.int64, device=self.device)
        args = [self._h, ctypes.byref(plan), self._rp(ct_in, (n_in, 2, L, n), "ct_in"),
                _ptr(x0, (n_in, n), "x0"), self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"),
                _ptr(r, (n_out, n), "r"), self._rp(out, (n_out, 2, L, n), "ct_out")]
        tail = [*_ws(workspace, ws_bytes, self.device), self._stream(stream)]
        if y0 is None:
            _check(self._f("he_conv2d")(*args, *tail))
        else:
            _check(self._f("he_conv2d_ex")(*args, _ptr(y0, (plan.M, plan.OH, plan.OW), "y0"), *tail))
        return out

    def online_workspace_bytes(self, plan: Plan) -> int:
        return int(lib().secn_he_conv2d_online_workspace(self._h, ctypes.byref(plan)))

    def he_conv2d_online(self, plan: Plan, ct_in: torch.Tensor, kernel: torch.Tensor,
                         x0: Optional[torch.Tensor] = None, r: Optional[torch.Tensor] = None,
                         out: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                         y0: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """secn_he_conv2d_online: weights in coefficient form (int64 [M][C][kh][kw]), transformed
        inside the call (online NTT preprocessing)."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        if out is None:
            out = self.empty(n_out, 2, L, n)
        need = self.online_workspace_bytes(plan)
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_online")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (n_in, 2, L, n), "ct_in"), _ptr(x0, (n_in, n), "x0"),
            _ptr(kernel, (plan.M, plan.C, plan.kh, plan.kw), "kernel"), _ptr(r, (n_out, n), "r"),
            self._rp(out, (n_out, 2, L, n), "ct_out"),
            _ptr(y0, (plan.M, plan.OH, plan.OW), "y0") if y0 is not None else None, wp, wn,
            self._stream(stream)))
        return out

    def he_conv2d_stage(self, stage: int, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor,
                        x0: Optional[torch.Tensor], r: Optional[torch.Tensor], out: torch.Tensor,
                        workspace: torch.Tensor, stream=None) -> torch.Tensor:
        """One launch group of secn_he_conv2d (0: share add + NTT, 1: MAC, 2: INTT + mask)."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        _check(self._f("he_conv2d_stage")(self._h, ctypes.byref(plan), stage,
                                          self._rp(ct_in, (n_in, 2, L, n), "ct_in"), _ptr(x0, (n_in, n), "x0"),
                                          self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), _ptr(r, (n_out, n), "r"),
                                          self._rp(out, (n_out, 2, L, n), "ct_out"),
                                          *_ws(workspace, self.workspace_bytes(plan), self.device),
                                          self._stream(stream)))
        return out

    def he_conv2d_stage_ex(self, stage: int, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor,
                           x0: Optional[torch.Tensor], r: Optional[torch.Tensor], out: torch.Tensor,
                           y0: Optional[torch.Tensor], workspace: torch.Tensor, stream=None) -> torch.Tensor:
        """secn_he_conv2d_stage_ex: one launch group, stage 2 also writing the share y0."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        _check(self._f("he_conv2d_stage_ex")(self._h, ctypes.byref(plan), stage,
                                             self._rp(ct_in, (n_in, 2, L, n), "ct_in"), _ptr(x0, (n_in, n), "x0"),
                                             self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), _ptr(r, (n_out, n), "r"),
                                             self._rp(out, (n_out, 2, L, n), "ct_out"),
                                             _ptr(y0, (plan.M, plan.OH, plan.OW), "y0") if y0 is not None else None,
                                             *_ws(workspace, self.workspace_bytes(plan), self.device),
                                             self._stream(stream)))
        return out

    # ---- device-drawn mask (reading R17) ----
    def mask_draw(self, gen: MaskGen, n_ct: int, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """secn_mask_draw: r int64 [n_ct][N] from the generator."""
        if out is None:
            out = torch.empty((n_ct, self.n), dtype=torch.int64, device=self.device)
        _check(lib().secn_mask_draw(self._h, ctypes.byref(gen), n_ct, _ptr(out, (n_ct, self.n), "r"),
                                    self._stream(stream)))
        return out

    def mask_encode(self, plan: Plan, r: Optional[torch.Tensor] = None, gen: Optional[MaskGen] = None,
                    out: Optional[torch.Tensor] = None, y0: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """secn_mask_encode: the encoded mask em [M*S][L][N] (residue dtype) from r or the generator,
        and y0 (int64 [M][OH][OW], optional) = -r mod t at the designated outputs."""
        shape = (plan.M * plan.S, self.L, self.n)
        if out is None:
            out = self.empty(*shape)
        _check(lib().secn_mask_encode(self._h, ctypes.byref(plan), _ptr(r, (plan.M * plan.S, self.n), "r"),
                                      ctypes.byref(gen) if gen is not None else None, self._rp(out, shape, "em"),
                                      _ptr(y0, (plan.M, plan.OH, plan.OW), "y0"), self._stream(stream)))
        return out

    def he_conv2d_em(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, em: torch.Tensor,
                     x0: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                     workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        """secn_he_conv2d_em: the layer with a mask encoded beforehand by mask_encode."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        if out is None:
            out = self.empty(n_out, 2, L, n)
        need = self.workspace_bytes(plan)
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_em")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (n_in, 2, L, n), "ct_in"), _ptr(x0, (n_in, n), "x0"),
            self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), self._rp(em, (n_out, L, n), "em"),
            self._rp(out, (n_out, 2, L, n), "ct_out"), wp, wn, self._stream(stream)))
        return out

    def he_conv2d_lwe_em(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, keep: int, em: torch.Tensor,
                         x0: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None, stream=None,
                         out: Optional[tuple] = None):
        """secn_he_conv2d_lwe_em: extracted outputs with a mask encoded beforehand."""
        L, n = self.L, self.n
        a, b = out if out is not None else (self.empty(plan.M * plan.S, keep, n), self.empty(plan.M, plan.OH, plan.OW, keep))
        need = int(lib().secn_he_conv2d_lwe_workspace(self._h, ctypes.byref(plan)))
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_lwe_em")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (plan.G * plan.S, 2, L, n), "ct_in"),
            _ptr(x0, (plan.G * plan.S, n), "x0"), self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"),
            self._rp(em, (plan.M * plan.S, L, n), "em"), keep, self._rp(a, (plan.M * plan.S, keep, n), "a_out"),
            self._rp(b, (plan.M, plan.OH, plan.OW, keep), "b_out"), wp, wn, self._stream(stream)))
        return a, b

    def gen_workspace_bytes(self, plan: Plan) -> int:
        return int(lib().secn_he_conv2d_gen_workspace(self._h, ctypes.byref(plan)))

    def he_conv2d_gen(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, gen: MaskGen,
                      x0: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                      y0: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                      stream=None) -> torch.Tensor:
        """secn_he_conv2d_gen: secn_he_conv2d_ex with the mask drawn on the device by `gen`."""
        L, n = self.L, self.n
        n_in, n_out = plan.G * plan.S, plan.M * plan.S
        if out is None:
            out = self.empty(n_out, 2, L, n)
        need = self.gen_workspace_bytes(plan)
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_gen")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (n_in, 2, L, n), "ct_in"), _ptr(x0, (n_in, n), "x0"),
            self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), ctypes.byref(gen),
            self._rp(out, (n_out, 2, L, n), "ct_out"), _ptr(y0, (plan.M, plan.OH, plan.OW), "y0"), wp, wn,
            self._stream(stream)))
        return out

    def he_conv2d_lwe_gen(self, plan: Plan, ct_in: torch.Tensor, w_ntt: torch.Tensor, keep: int, gen: MaskGen,
                          x0: Optional[torch.Tensor] = None, y0: Optional[torch.Tensor] = None,
                          workspace: Optional[torch.Tensor] = None, stream=None, out: Optional[tuple] = None):
        """secn_he_conv2d_lwe_gen: extracted outputs with the mask drawn on the device."""
        L, n = self.L, self.n
        a, b = out if out is not None else (self.empty(plan.M * plan.S, keep, n), self.empty(plan.M, plan.OH, plan.OW, keep))
        need = int(lib().secn_he_conv2d_lwe_gen_workspace(self._h, ctypes.byref(plan)))
        if workspace is None:
            workspace = torch.empty((need + 7) // 8, dtype=torch.int64, device=self.device)
        wp, wn = _ws(workspace, need, self.device)
        _check(self._f("he_conv2d_lwe_gen")(
            self._h, ctypes.byref(plan), self._rp(ct_in, (plan.G * plan.S, 2, L, n), "ct_in"),
            _ptr(x0, (plan.G * plan.S, n), "x0"), self._rp(w_ntt, (plan.M, plan.G, L, n), "w_ntt"), ctypes.byref(gen),
            keep, self._rp(a, (plan.M * plan.S, keep, n), "a_out"), self._rp(b, (plan.M, plan.OH, plan.OW, keep), "b_out"),
            _ptr(y0, (plan.M, plan.OH, plan.OW), "y0"), wp, wn, self._stream(stream)))
        return a, b

    def extract_share(self, plan: Plan, r: torch.Tensor, out: Optional[torch.Tensor] = None,
                      stream=None) -> torch.Tensor:
        shape = (plan.M, plan.OH, plan.OW)
        if out is None:
            out = torch.empty(shape, dtype=torch.int64, device=self.device)
        _check(lib().secn_extract_share(self._h, ctypes.byref(plan), _ptr(r, (plan.M * plan.S, self.n), "r"),
                                        _ptr(out, shape, "y0"), self._stream(stream)))
        return out
