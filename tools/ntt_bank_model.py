"""Shared-memory bank-conflict model of the NTT rounds (32 banks x 4 bytes): for every radix-16
round of the forward (CT) and inverse (GS) transform at N = 2^12..2^14 and both word sizes, the
worst number of distinct 128-byte lines one bank serves in a warp-wide scalar access, under the
padded layout of the one-CTA-per-poly kernels (phys(e) = e + e/16) and the TMA 128-byte swizzle
of k_ntt_tma (stage_swz). Contiguous-task rounds of k_ntt_tma use 16-byte vector accesses,
checked per 8-thread phase. Usage: python tools/ntt_bank_model.py"""


def swz(e, lw):
    return e ^ (((e >> (7 - lw)) & 7) << (4 - lw))


def phys(e):
    return e + (e >> 4)


def rounds(logn, gs):
    out, s = [], 0
    while s < logn:
        k = min(4, logn - s)
        logb, logd = (s + k, s) if gs else (logn - s, logn - s - k)
        out.append((s, k, logb, logd))
        s += k
    return out


def addr(tau, i, logb, logd):
    return ((tau >> logd) << logb) + (tau & ((1 << logd) - 1)) + (i << logd)


def degree(words, lw):
    banks = {}
    for a in words:
        byte = a << lw
        for b in range((1 << lw) // 4):
            banks.setdefault(((byte >> 2) + b) % 32, set()).add(byte >> 7)
    return max(len(v) for v in banks.values())


def vector_degree(words, lw):
    """16-byte accesses, served 8 threads per phase: worst number of threads of a phase that hit
    the same 16-byte bank group"""
    worst = 1
    for p in range(0, len(words), 8):
        groups = [((a << lw) >> 4) % 8 for a in words[p:p + 8]]
        worst = max(worst, max(groups.count(g) for g in groups))
    return worst


for logn in (12, 13, 14):
    t = (1 << logn) // 16
    for lw, name in ((2, "u32"), (3, "u64")):
        for gs in (False, True):
            res = []
            for (s, k, logb, logd) in rounds(logn, gs):
                gk, nt = 1 << k, 16 // (1 << k)
                sw = pad = vec = 1
                for w in range(t // 32):
                    for kk in range(nt):
                        for i in range(gk):
                            a = [addr(32 * w + l + kk * t, i, logb, logd) for l in range(32)]
                            sw = max(sw, degree([swz(x, lw) for x in a], lw))
                            pad = max(pad, degree([phys(x) for x in a], lw))
                        if logd == 0 and gk * (1 << lw) >= 16:
                            for v in range(gk * (1 << lw) // 16):
                                a = [addr(32 * w + l + kk * t, v * (16 >> lw), logb, logd) for l in range(32)]
                                vec = max(vec, vector_degree([swz(x, lw) for x in a], lw))
                tag = f" vec16={vec}" if logd == 0 and gk * (1 << lw) >= 16 else ""
                res.append(f"levels {s}-{s + k - 1}: pad {pad} swz {sw}{tag}")
            print(f"N=2^{logn} {name} {'GS' if gs else 'CT'}: " + "; ".join(res))
