"""Cheetah coefficient packing for HE convolution -- oracle side (test infrastructure only).

The paper states the property, not the formulas: Cheetah "encodes messages directly into
the coefficients of the polynomials ... placed strategically within the polynomials such
that one vector dot product is computed with a single polynomial multiplication. This
strategy results in a sparse output with very few coefficients containing the actual
result" (§2.3; §6.1). SPEC.md:626 adds "input at index
c*HW + h*W + w; kernel mirrored". The formulas below are DESIGN.md reading R6/R7/R8; they are
pinned by the end-to-end test decrypt(server(Enc(x))) = conv(x, K) mod 2^t.

Geometry
    Xe      effective input: zero-padded by `pad`, and for a 1x1 kernel with stride > 1
            pre-decimated to Xe[c, i, j] = Xpad[c, i*stride, j*stride] (reading R7, decim = 1);
            for a larger kernel with stride s > 1 optionally split into its s^2 polyphase
            components (reading R7b, decim = 2): Ce = C s^2 channels
                Xe[(c s + u) s + v, i, j] = Xpad[c, i s + u, j s + v],
            and the kernel likewise, Ke[m, (c s + u) s + v, a, b] = K[m, c, s a + u, s b + v]
            (0 where s a + u >= kh or s b + v >= kw), of size khe x kwe = ceil(kh/s) x ceil(kw/s).
            Then y[oy, ox] = sum_{c',a,b} Xe[c', oy+a, ox+b] Ke[m, c', a, b] -- a stride-1
            correlation whose every window position is an output (no strided designation).
    Ce, khe, kwe   the channel count and kernel extent the windows use (C, kh, kw unless decim = 2)
    Hp, Wp  extent of Xe;  Ph, Pw = number of stride-1 window positions that must be covered
    window  Cw channels x Hw rows x Ww cols per polynomial, Cw*Hw*Ww <= N
    G       = ceil(Ce / Cw) channel groups;  S = nbh * nbw spatial blocks
    O       = (Cw-1)*Hw*Ww + (khe-1)*Ww + (kwe-1)

    input poly (g, s), s = bh*nbw + bw, origin (h0, w0) = (bh*(Hw-khe+1), bw*(Ww-kwe+1)):
        coeff[c*Hw*Ww + i*Ww + j] = Xe[g*Cw + c, h0+i, w0+j]      (0 outside Xe)
    kernel poly (m, g):
        coeff[O - c*Hw*Ww - l*Ww - l'] = Ke[m, g*Cw + c, l, l']
    output poly (m, s), designated coefficient O + i*Ww + j (0 <= i <= Hw-khe, 0 <= j <= Ww-kwe)
        = sum_{c,l,l'} Xe[c, h0+i+l, w0+j+l'] Ke[m, c, l, l']  = stride-1 output at (h0+i, w0+j)
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Plan:
    C: int
    H: int
    W: int
    M: int
    kh: int
    kw: int
    stride: int
    pad: int
    OH: int
    OW: int
    decim: int
    Hp: int
    Wp: int
    Cw: int
    Hw: int
    Ww: int
    G: int
    S: int
    nbh: int
    nbw: int
    O: int

    @property
    def ps(self) -> int:
        """polyphase factor (reading R7b): the stride when decim = 2, else 1"""
        return self.stride if self.decim == 2 else 1

    @property
    def Ce(self) -> int:
        return self.C * self.ps * self.ps

    @property
    def khe(self) -> int:
        return -(-self.kh // self.ps)

    @property
    def kwe(self) -> int:
        return -(-self.kw // self.ps)


def _geometry(C, H, W, kh, kw, stride, pad, poly=False):
    """(OH, OW, decim, Hp, Wp, Ph, Pw); poly requests the polyphase split (reading R7b), which
    applies to strided kernels larger than 1x1 only."""
    OH = (H + 2 * pad - kh) // stride + 1
    OW = (W + 2 * pad - kw) // stride + 1
    decim = 1 if (kh == 1 and kw == 1 and stride > 1) else 0
    if poly:
        if decim or stride == 1:
            raise ValueError("polyphase packing needs stride > 1 and a kernel larger than 1x1")
        decim = 2
    if decim == 1:
        Hp, Wp, Ph, Pw = OH, OW, OH, OW
    elif decim == 2:
        Hp, Wp, Ph, Pw = -(-(H + 2 * pad) // stride), -(-(W + 2 * pad) // stride), OH, OW
    else:
        Hp, Wp = H + 2 * pad, W + 2 * pad
        Ph, Pw = (OH - 1) * stride + 1, (OW - 1) * stride + 1
    return OH, OW, decim, Hp, Wp, Ph, Pw


def plan_conv(C, H, W, M, kh, kw, stride=1, pad=0, n=4096, L=2, Hw=None, Ww=None, poly=False,
              rule="bytes") -> Plan:
    """Reading R6 (rule="bytes"): enumerate Hw in [khe, Hp], Ww in [kwe, Wp] with Hw*Ww <= N, take
    Cw = min(Ce, N // (Hw*Ww)), and minimise the algorithmic bytes
        8*L*N*(2*G*S + M*G + 2*M*S) + 8*N*M*S
    tie-breaking on fewer M*G*S products, then larger Hw, then larger Ww.
    An explicit (Hw, Ww) is validated and used instead. poly: the polyphase split of reading
    R7b (strided kernels larger than 1x1). L is the number of 8-byte words per coefficient of one
    ciphertext component (the limb count for 64-bit limbs, half of it for 32-bit limbs).
    rule="time": reading R6b, see plan_conv_time (Hw, Ww, poly are then ignored)."""
    if rule == "time":
        return plan_conv_time(C, H, W, M, kh, kw, stride, pad, n, L)
    if rule != "bytes":
        raise ValueError(f"unknown plan rule {rule!r}")
    OH, OW, decim, Hp, Wp, Ph, Pw = _geometry(C, H, W, kh, kw, stride, pad, poly)
    if OH <= 0 or OW <= 0 or kh * kw > n:
        raise ValueError("unsupported shape")
    ps = stride if decim == 2 else 1
    Ce, khe, kwe = C * ps * ps, -(-kh // ps), -(-kw // ps)
    best = None
    cands = [(Hw, Ww)] if Hw is not None else [(a, b) for a in range(khe, Hp + 1) for b in range(kwe, Wp + 1)]
    for a, b in cands:
        if a < khe or b < kwe or a * b > n or a > Hp or b > Wp:
            continue
        Cw = min(Ce, n // (a * b))
        G = -(-Ce // Cw)
        nbh = -(-Ph // (a - khe + 1))
        nbw = -(-Pw // (b - kwe + 1))
        S = nbh * nbw
        cost = 8 * L * n * (2 * G * S + M * G + 2 * M * S) + 8 * n * M * S
        key = (cost, M * G * S, -a, -b)
        if best is None or key < best[0]:
            best = (key, a, b, Cw, G, S, nbh, nbw)
    if best is None:
        raise ValueError("unsupported shape: no window fits N")
    _, a, b, Cw, G, S, nbh, nbw = best
    O = (Cw - 1) * a * b + (khe - 1) * b + (kwe - 1)
    return Plan(C, H, W, M, kh, kw, stride, pad, OH, OW, decim, Hp, Wp, Cw, a, b, G, S, nbh, nbw, O)


def plan_conv_time(C, H, W, M, kh, kw, stride=1, pad=0, n=4096, L=2) -> Plan:
    """Reading R6b (the window rule the product library applies by default): among
    every valid window -- plain and, for a strided kernel larger than 1x1, polyphase (reading R7b)
    -- with G <= 30 (G <= 32 if no window has G <= 30), minimise the modelled device time in ns
        t = 2 lp (13 M S + 1.3 M S G + 6 G S) + 0.3 bytes / 6450,   lp = 2 L N / 4096
    (bytes = the R6 algorithmic bytes). Windows are scanned plain before polyphase, Hw then Ww
    ascending; a window replaces the best so far if its t is smaller by a relative 1e-12, or
    equal within 1e-12 and it has fewer bytes, or the same bytes and a larger Hw, then Ww. The
    packing (and so every result) is exact for any window; the rule only picks a fast one."""
    can_poly = stride > 1 and not (kh == 1 and kw == 1)
    lp = 2.0 * L * n / 4096.0
    for gmax in (30, 32):
        best = None
        best_t = best_cost = 0
        for poly in ((False, True) if can_poly else (False,)):
            OH, OW, decim, Hp, Wp, Ph, Pw = _geometry(C, H, W, kh, kw, stride, pad, poly)
            ps = stride if decim == 2 else 1
            khe, kwe = -(-kh // ps), -(-kw // ps)
            for a in range(khe, Hp + 1):
                for b in range(kwe, Wp + 1):
                    if a * b > n:
                        break
                    p = plan_conv(C, H, W, M, kh, kw, stride, pad, n, L, Hw=a, Ww=b, poly=poly)
                    if p.G > gmax:
                        continue
                    G, S = p.G, p.S
                    cost = 8 * L * n * (2 * G * S + M * G + 2 * M * S) + 8 * n * M * S
                    ms, gs = float(M * S), float(G * S)
                    t = 2.0 * lp * (13.0 * ms + 1.3 * ms * float(G) + 6.0 * gs) + 0.3 * float(cost) / 6450.0
                    if (best is None or t < best_t * (1 - 1e-12) or
                            (t <= best_t * (1 + 1e-12) and
                             (cost < best_cost or (cost == best_cost and (a > best.Hw or (a == best.Hw and b > best.Ww)))))):
                        best, best_t, best_cost = p, t, cost
        if best is not None:
            return best
    raise ValueError("unsupported shape: no window fits N")


def effective_input(x: np.ndarray, p: Plan) -> np.ndarray:
    """Zero-pad the input share (C,H,W); for decimated 1x1/stride>1 plans subsample it, for
    polyphase plans split it into Xe[(c s + u) s + v, i, j] = Xpad[c, i s + u, j s + v]."""
    xp = np.zeros((p.C, p.H + 2 * p.pad, p.W + 2 * p.pad), dtype=np.uint64)
    xp[:, p.pad:p.pad + p.H, p.pad:p.pad + p.W] = x
    if p.decim == 1:
        xp = xp[:, ::p.stride, ::p.stride][:, :p.OH, :p.OW]
    elif p.decim == 2:
        s = p.stride
        xe = np.zeros((p.Ce, p.Hp, p.Wp), dtype=np.uint64)
        for c in range(p.C):
            for u in range(s):
                for v in range(s):
                    comp = xp[c, u::s, v::s]
                    xe[(c * s + u) * s + v, :comp.shape[0], :comp.shape[1]] = comp
        xp = xe
    return np.ascontiguousarray(xp)


def pack_input(x: np.ndarray, p: Plan, n: int) -> np.ndarray:
    """Input share (C,H,W) -> polys [G*S][N] (index g*S+s)."""
    xe = effective_input(x, p)
    out = np.zeros((p.G * p.S, n), dtype=np.uint64)
    for g in range(p.G):
        for bh in range(p.nbh):
            for bw in range(p.nbw):
                s = bh * p.nbw + bw
                h0, w0 = bh * (p.Hw - p.khe + 1), bw * (p.Ww - p.kwe + 1)
                for c in range(p.Cw):
                    cc = g * p.Cw + c
                    if cc >= p.Ce:
                        break
                    for i in range(p.Hw):
                        if h0 + i >= p.Hp:
                            break
                        row = xe[cc, h0 + i, w0:min(w0 + p.Ww, p.Wp)]
                        base = c * p.Hw * p.Ww + i * p.Ww
                        out[g * p.S + s, base:base + row.size] = row
    return out


def effective_kernel(K: np.ndarray, p: Plan) -> np.ndarray:
    """Kernel (M,C,kh,kw) -> (M,Ce,khe,kwe): itself, or its polyphase split (reading R7b)."""
    if p.decim != 2:
        return K
    s = p.stride
    Ke = np.zeros((K.shape[0], p.Ce, p.khe, p.kwe), dtype=K.dtype)
    for c in range(p.C):
        for u in range(s):
            for v in range(s):
                comp = K[:, c, u::s, v::s]
                Ke[:, (c * s + u) * s + v, :comp.shape[1], :comp.shape[2]] = comp
    return Ke


def kernel_polys(K: np.ndarray, p: Plan, n: int) -> np.ndarray:
    """Kernel (M,C,kh,kw) values < 2^t -> raw mirrored plaintext polys [M][G][N] (not lifted)."""
    Ke = effective_kernel(K, p)
    out = np.zeros((p.M, p.G, n), dtype=np.uint64)
    for m in range(p.M):
        for g in range(p.G):
            for c in range(p.Cw):
                cc = g * p.Cw + c
                if cc >= p.Ce:
                    break
                for l in range(p.khe):
                    for l2 in range(p.kwe):
                        out[m, g, p.O - c * p.Hw * p.Ww - l * p.Ww - l2] = Ke[m, cc, l, l2]
    return out


def sparse(polys: np.ndarray):
    """[M][G][N] -> (koff, kidx, kval) CSR over the M*G polys, nonzero coefficients only."""
    MG = polys.shape[0] * polys.shape[1]
    flat = polys.reshape(MG, -1)
    koff = np.zeros(MG + 1, dtype=np.uint64)
    idx, val = [], []
    for r in range(MG):
        nz = np.nonzero(flat[r])[0]
        idx.append(nz.astype(np.uint32))
        val.append(flat[r, nz])
        koff[r + 1] = koff[r] + nz.size
    kidx = np.concatenate(idx) if idx else np.zeros(0, np.uint32)
    kval = np.concatenate(val) if val else np.zeros(0, np.uint64)
    return koff, np.ascontiguousarray(kidx), np.ascontiguousarray(kval)


def designated_map(p: Plan):
    """Arrays (s_idx, coef_idx) of shape (OH, OW): output (oy, ox) of channel m is coefficient
    coef_idx[oy, ox] of output poly (m, s_idx[oy, ox])."""
    sh = 1 if p.decim else p.stride
    oy, ox = np.meshgrid(np.arange(p.OH), np.arange(p.OW), indexing="ij")
    py, px = oy * sh, ox * sh
    bh, i = py // (p.Hw - p.khe + 1), py % (p.Hw - p.khe + 1)
    bw, j = px // (p.Ww - p.kwe + 1), px % (p.Ww - p.kwe + 1)
    return bh * p.nbw + bw, p.O + i * p.Ww + j


def extract(polys: np.ndarray, p: Plan) -> np.ndarray:
    """polys [M*S][N] (values mod t) -> y [M][OH][OW] at the designated coefficients."""
    s_idx, coef = designated_map(p)
    P = polys.reshape(p.M, p.S, -1)
    return P[:, s_idx, coef]
