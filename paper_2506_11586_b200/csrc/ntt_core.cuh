// Shared-memory negacyclic NTT core: NP limb-polys of the same limb per CTA (they share every
// twiddle), N = 2^LOGN, T = N/16 threads, 16 words per poly per thread in registers;
// parameterised by an arithmetic policy A (modarith.cuh).
//
// Forward = Cooley-Tukey with psi^brv twiddles, natural order in, bit-reversed order out
// (reading R4: entry k holds a(psi^(2 brv(k)+1))); inverse = Gentleman-Sande with psi^-brv
// twiddles and N^-1 folded into the last level (App. C.1).
//
// A "round" performs K <= 4 consecutive stages in registers: the 2^K elements of a task are
// blk*B + off + i*D (i < 2^K) and every thread owns 16/2^K tasks. Rounds exchange data through
// shared memory in a padded layout (phys) that makes every round's addresses immediate offsets.
#pragma once
#include <cstdint>

#include "modarith.cuh"
#include "tma.cuh"

namespace secn {

// Shared-memory layout: word e lives at phys(e) = e + (e >> 4) (one pad word per 16). Every
// round's task pattern then maps to phys(base) + const, so addresses are immediate offsets from
// one per-task base register, and 64-bit words are bank-conflict free in every pattern (16 lanes
// hit 16 distinct bank pairs); 32-bit words see at most 2-way conflicts on the contiguous
// patterns. A buffer of N words needs N + N/16 words (smem_words); poly p of a CTA starts at
// p * smem_words.
__host__ __device__ __forceinline__ constexpr uint32_t phys(uint32_t e) { return e + (e >> 4); }
template <int LOGN>
__host__ __device__ constexpr int smem_words() { return (1 << LOGN) + (1 << LOGN) / 16; }

template <int LOGN, int S0>
struct CtRound {
  static constexpr int K = (LOGN - S0) >= 4 ? 4 : (LOGN - S0);
  static constexpr int GK = 1 << K, NT = 16 / GK, T = (1 << LOGN) / 16;
  static constexpr int logB = LOGN - S0, logD = logB - K;
  __device__ static __forceinline__ uint32_t blk(int k) { return (threadIdx.x + k * T) >> logD; }
  __device__ static __forceinline__ uint32_t addr(int k, int i) {
    const uint32_t tau = threadIdx.x + k * T;
    return ((tau >> logD) << logB) + (tau & ((1u << logD) - 1)) + (i << logD);
  }
  // phys(addr(k, i)) = pbase(k) + poff(i) (see phys)
  __device__ static __forceinline__ uint32_t pbase(int k) { return phys(addr(k, 0)); }
  __host__ __device__ static constexpr uint32_t poff(int i) { return (i << logD) + ((i << logD) >> 4); }
};

template <int LOGN, int L0>
struct GsRound {
  static constexpr int K = (LOGN - L0) >= 4 ? 4 : (LOGN - L0);
  static constexpr int GK = 1 << K, NT = 16 / GK, T = (1 << LOGN) / 16;
  static constexpr int logB = L0 + K, logD = L0;
  __device__ static __forceinline__ uint32_t blk(int k) { return (threadIdx.x + k * T) >> logD; }
  __device__ static __forceinline__ uint32_t addr(int k, int i) {
    const uint32_t tau = threadIdx.x + k * T;
    return ((tau >> logD) << logB) + (tau & ((1u << logD) - 1)) + (i << logD);
  }
  __device__ static __forceinline__ uint32_t pbase(int k) { return phys(addr(k, 0)); }
  __host__ __device__ static constexpr uint32_t poff(int i) { return (i << logD) + ((i << logD) >> 4); }
};

// shared-memory round trip of the x[NP][16] register block of round R
template <class R, class W, int NP, int LOGN>
__device__ __forceinline__ void round_load(W (&x)[NP][16], const W* sm) {
#pragma unroll
  for (int k = 0; k < R::NT; ++k) {
    const uint32_t b = R::pbase(k);
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int i = 0; i < R::GK; ++i) x[pp][k * R::GK + i] = sm[pp * smem_words<LOGN>() + b + R::poff(i)];
  }
}

template <class R, class W, int NP, int LOGN>
__device__ __forceinline__ void round_store(const W (&x)[NP][16], W* sm) {
#pragma unroll
  for (int k = 0; k < R::NT; ++k) {
    const uint32_t b = R::pbase(k);
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int i = 0; i < R::GK; ++i) sm[pp * smem_words<LOGN>() + b + R::poff(i)] = x[pp][k * R::GK + i];
  }
}

// Global-memory load / store of a round whose tasks are contiguous (logD == 0: the GS round at
// level 0, the last CT round): task k's GK words are consecutive, moved as 16-byte (or narrower)
// vectors. The warp-level access is not coalesced per instruction, but every thread moves whole
// 32-byte sectors, so the sectors are used in full across the round's vector instructions.
template <class W, int VW>
struct Vec;
template <> struct Vec<uint32_t, 4> { using T = uint4; };
template <> struct Vec<uint32_t, 2> { using T = uint2; };
template <> struct Vec<uint32_t, 1> { using T = uint32_t; };
template <> struct Vec<uint64_t, 2> { using T = ulonglong2; };
template <> struct Vec<uint64_t, 1> { using T = uint64_t; };

template <class R, class W, int NP>
__device__ __forceinline__ void round_gload(W (&x)[NP][16], const W* const (&src)[NP]) {
  static_assert(R::logD == 0, "contiguous tasks only");
  constexpr int VW = (int)(16 / sizeof(W)) < R::GK ? (int)(16 / sizeof(W)) : R::GK;
  using V = typename Vec<W, VW>::T;
#pragma unroll
  for (int k = 0; k < R::NT; ++k) {
    const uint32_t b = R::addr(k, 0);
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int v = 0; v < R::GK / VW; ++v) {
        const V t = *reinterpret_cast<const V*>(src[pp] + b + v * VW);
        const W* tw = reinterpret_cast<const W*>(&t);
#pragma unroll
        for (int u = 0; u < VW; ++u) x[pp][k * R::GK + v * VW + u] = tw[u];
      }
  }
}

template <class R, class W, int NP>
__device__ __forceinline__ void round_gstore(const W (&x)[NP][16], W* const (&dst)[NP]) {
  static_assert(R::logD == 0, "contiguous tasks only");
  constexpr int VW = (int)(16 / sizeof(W)) < R::GK ? (int)(16 / sizeof(W)) : R::GK;
  using V = typename Vec<W, VW>::T;
#pragma unroll
  for (int k = 0; k < R::NT; ++k) {
    const uint32_t b = R::addr(k, 0);
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int v = 0; v < R::GK / VW; ++v) {
        V t;
        W* tw = reinterpret_cast<W*>(&t);
#pragma unroll
        for (int u = 0; u < VW; ++u) tw[u] = x[pp][k * R::GK + v * VW + u];
        *reinterpret_cast<V*>(dst[pp] + b + v * VW) = t;
      }
  }
}

// The dense swizzled layout of TMA's 128-byte swizzle: word e of a poly at stage_swz(e) (the
// 16-byte chunk index XOR the 128-byte row index mod 8, relative to a 1024-byte-aligned base;
// with a 16-byte-aligned base the bank pattern is the same up to a rotation).
template <class W>
__host__ __device__ __forceinline__ constexpr uint32_t stage_swz(uint32_t e) {
  constexpr int lw = sizeof(W) == 4 ? 2 : 3;  // log2 of the word size
  return e ^ (((e >> (7 - lw)) & 7) << (4 - lw));
}

// The last CT round's words (contiguous tasks) to global memory through shared memory, so that
// each warp store instruction covers 512 contiguous bytes instead of 16 bytes every 64 (which
// half-fills every 32-byte sector per instruction). sm holds >= NP * N words and every thread
// has finished reading it (the caller's barrier).
template <class R, class W, int NP, int LOGN>
__device__ __forceinline__ void round_gstore_coalesced(const W (&x)[NP][16], W* sm, W* const (&dst)[NP]) {
  constexpr int N = 1 << LOGN, VW = 16 / (int)sizeof(W);
  static_assert(R::logD == 0 && R::GK >= VW, "contiguous tasks of whole 16-byte chunks");
#pragma unroll
  for (int k = 0; k < R::NT; ++k)
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int v = 0; v < R::GK / VW; ++v) {
        uint4 t;
        W* tv = reinterpret_cast<W*>(&t);
#pragma unroll
        for (int u = 0; u < VW; ++u) tv[u] = x[pp][k * R::GK + v * VW + u];
        *reinterpret_cast<uint4*>(sm + pp * N + stage_swz<W>(R::addr(k, v * VW))) = t;
      }
  __syncthreads();
#pragma unroll
  for (int pp = 0; pp < NP; ++pp)
#pragma unroll
    for (int v = 0; v < 16 / VW; ++v) {
      const uint32_t ch = threadIdx.x + v * R::T;  // 16-byte chunk: 16 per thread per poly
      *reinterpret_cast<uint4*>(dst[pp] + ch * VW) = *reinterpret_cast<const uint4*>(sm + pp * N + stage_swz<W>(ch * VW));
    }
}

// ------------------------------------------------------------------------------------------
// Cooley-Tukey: stages S0 .. S0+K-1 (stage s: 2^s groups, group i uses psi^brv(2^s + i)).
// Twiddles of one round are gathered into registers before the round's barrier so their load
// latency overlaps it: task k, stage p, group u -> tws[k * (GK - 1) + (1 << p) - 1 + u] (<= 15).
template <class A, int LOGN, int S0>
__device__ __forceinline__ void ct_twiddles(typename A::Tw (&tws)[15], const typename A::Tw* __restrict__ tw) {
  using R = CtRound<LOGN, S0>;
  const uint64_t pol = policy_evict_last();  // the tables are reused by every layer: keep them in L2
#pragma unroll
  for (int p = 0; p < R::K; ++p)
#pragma unroll
    for (int k = 0; k < R::NT; ++k)
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < (1 << p))
          tws[k * (R::GK - 1) + (1 << p) - 1 + u] = ldg_hint(&tw[(1u << (S0 + p)) + (R::blk(k) << p) + u], pol);
}

template <class A, int LOGN, int S0, int NP>
__device__ __forceinline__ void ct_compute(typename A::W (&x)[NP][16], const typename A::Tw (&tws)[15],
                                           typename A::W q, typename A::W qb) {
  using R = CtRound<LOGN, S0>;
#pragma unroll
  for (int p = 0; p < R::K; ++p) {
    const int half = R::GK >> (p + 1);
#pragma unroll
    for (int k = 0; k < R::NT; ++k) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < (1 << p)) {
          const typename A::Tw w = tws[k * (R::GK - 1) + (1 << p) - 1 + u];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < half) {
              const int a = k * R::GK + u * (R::GK >> p) + i;
#pragma unroll
              for (int pp = 0; pp < NP; ++pp) A::ct(x[pp][a], x[pp][a + half], w, q, qb);
            }
          }
        }
      }
    }
  }
}

// S0 of the last CT round
template <int LOGN, int S0 = 0>
struct CtLast {
  static constexpr int value =
      (S0 + CtRound<LOGN, S0>::K >= LOGN) ? S0 : CtLast<LOGN, S0 + CtRound<LOGN, S0>::K>::value;
};
template <int LOGN>
struct CtLast<LOGN, LOGN> {
  static constexpr int value = LOGN;
};

// Rounds S0.. up to (not including) the last one, each: gather twiddles, barrier (the previous
// round's stores), smem -> regs -> smem. The caller runs the last round.
template <class A, int LOGN, int S0, int NP>
__device__ __forceinline__ void ct_rounds_smem_but_last(typename A::W* sm, const typename A::Tw* __restrict__ tw,
                                                        typename A::W q, typename A::W qb) {
  using R = CtRound<LOGN, S0>;
  if constexpr (S0 + R::K < LOGN) {
    typename A::Tw tws[15];
    ct_twiddles<A, LOGN, S0>(tws, tw);
    __syncthreads();
    typename A::W x[NP][16];
    round_load<R, typename A::W, NP, LOGN>(x, sm);
    ct_compute<A, LOGN, S0, NP>(x, tws, q, qb);
    round_store<R, typename A::W, NP, LOGN>(x, sm);
    ct_rounds_smem_but_last<A, LOGN, S0 + R::K, NP>(sm, tw, q, qb);
  }
}

// ------------------------------------------------------------------------------------------
// Gentleman-Sande: levels L0 .. L0+K-1 (level l: half-distance 2^l, N/2^(l+1) groups, group i
// uses psi^-brv(N/2^(l+1) + i)); the last level (l = LOGN-1) multiplies by N^-1 instead.
// Twiddles: task k, level p, group gi -> tws[k * (GK - 1) + GK - (GK >> p) + gi].
template <class A, int LOGN, int L0>
__device__ __forceinline__ void gs_twiddles(typename A::Tw (&tws)[15], const typename A::Tw* __restrict__ tw) {
  using R = GsRound<LOGN, L0>;
  const uint64_t pol = policy_evict_last();
#pragma unroll
  for (int p = 0; p < R::K; ++p) {
    if (L0 + p == LOGN - 1) continue;
    const uint32_t h = (1u << LOGN) >> (L0 + p + 1);
#pragma unroll
    for (int k = 0; k < R::NT; ++k)
#pragma unroll
      for (int gi = 0; gi < 8; ++gi)
        if (gi < (R::GK >> (p + 1)))
          tws[k * (R::GK - 1) + R::GK - (R::GK >> p) + gi] = ldg_hint(&tw[h + (R::blk(k) << (R::K - p - 1)) + gi], pol);
  }
}

template <class A, int LOGN, int L0, int NP>
__device__ __forceinline__ void gs_compute(typename A::W (&x)[NP][16], const typename A::Tw (&tws)[15],
                                           typename A::W q, typename A::W qb, typename A::Tw ninv,
                                           typename A::Tw wlast) {
  using R = GsRound<LOGN, L0>;
#pragma unroll
  for (int p = 0; p < R::K; ++p) {
    const int dist = 1 << p;
    if (L0 + p == LOGN - 1) {  // compile-time after unrolling
#pragma unroll
      for (int k = 0; k < R::NT; ++k)
#pragma unroll
        for (int i = 0; i < R::GK; ++i) {
          if (i & dist) continue;
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            const typename A::W u = x[pp][k * R::GK + i], v = x[pp][k * R::GK + i + dist];
            x[pp][k * R::GK + i] = A::mul4(u + v, ninv, q);
            x[pp][k * R::GK + i + dist] = A::mul4(u - v + qb, wlast, q);
          }
        }
    } else {
#pragma unroll
      for (int k = 0; k < R::NT; ++k) {
#pragma unroll
        for (int gi = 0; gi < 8; ++gi) {
          if (gi < (R::GK >> (p + 1))) {
            const typename A::Tw w = tws[k * (R::GK - 1) + R::GK - (R::GK >> p) + gi];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < dist) {
                const int a = k * R::GK + gi * (2 * dist) + i;
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) A::gs(x[pp][a], x[pp][a + dist], w, q, qb);
              }
            }
          }
        }
      }
    }
  }
}

// All GS rounds except the last one, each: gather twiddles, barrier, smem -> regs -> smem. The
// caller gathers the last round's twiddles and places the last barrier.
template <class A, int LOGN, int L0, int NP>
__device__ __forceinline__ void gs_rounds_smem_but_last(typename A::W* sm, const typename A::Tw* __restrict__ tw,
                                                        typename A::W q, typename A::W qb, typename A::Tw ninv,
                                                        typename A::Tw wlast) {
  using R = GsRound<LOGN, L0>;
  if constexpr (L0 + R::K < LOGN) {
    typename A::Tw tws[15];
    gs_twiddles<A, LOGN, L0>(tws, tw);
    __syncthreads();
    typename A::W x[NP][16];
    round_load<R, typename A::W, NP, LOGN>(x, sm);
    gs_compute<A, LOGN, L0, NP>(x, tws, q, qb, ninv, wlast);
    round_store<R, typename A::W, NP, LOGN>(x, sm);
    gs_rounds_smem_but_last<A, LOGN, L0 + R::K, NP>(sm, tw, q, qb, ninv, wlast);
  }
}

// The same levels with each butterfly group's twiddle loaded at its use instead of gathered into
// registers first (15 pairs = 60 registers for 64-bit words): for kernels whose register budget
// cannot hold them (64-bit words at N = 2^14, 1024 threads per CTA).
template <class A, int LOGN, int L0, int NP>
__device__ __forceinline__ void gs_compute_ld(typename A::W (&x)[NP][16], const typename A::Tw* __restrict__ tw,
                                              typename A::W q, typename A::W qb, typename A::Tw ninv,
                                              typename A::Tw wlast) {
  using R = GsRound<LOGN, L0>;
#pragma unroll
  for (int p = 0; p < R::K; ++p) {
    const int dist = 1 << p;
    if (L0 + p == LOGN - 1) {
#pragma unroll
      for (int k = 0; k < R::NT; ++k)
#pragma unroll
        for (int i = 0; i < R::GK; ++i) {
          if (i & dist) continue;
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            const typename A::W u = x[pp][k * R::GK + i], v = x[pp][k * R::GK + i + dist];
            x[pp][k * R::GK + i] = A::mul4(u + v, ninv, q);
            x[pp][k * R::GK + i + dist] = A::mul4(u - v + qb, wlast, q);
          }
        }
    } else {
      const uint32_t h = (1u << LOGN) >> (L0 + p + 1);
#pragma unroll
      for (int k = 0; k < R::NT; ++k) {
#pragma unroll
        for (int gi = 0; gi < 8; ++gi) {
          if (gi < (R::GK >> (p + 1))) {
            const typename A::Tw w = tw[h + (R::blk(k) << (R::K - p - 1)) + gi];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i < dist) {
                const int a = k * R::GK + gi * (2 * dist) + i;
#pragma unroll
                for (int pp = 0; pp < NP; ++pp) A::gs(x[pp][a], x[pp][a + dist], w, q, qb);
              }
            }
          }
        }
      }
    }
  }
}

template <class A, int LOGN, int L0, int NP>
__device__ __forceinline__ void gs_rounds_smem_but_last_ld(typename A::W* sm, const typename A::Tw* __restrict__ tw,
                                                           typename A::W q, typename A::W qb, typename A::Tw ninv,
                                                           typename A::Tw wlast) {
  using R = GsRound<LOGN, L0>;
  if constexpr (L0 + R::K < LOGN) {
    __syncthreads();
    typename A::W x[NP][16];
    round_load<R, typename A::W, NP, LOGN>(x, sm);
    gs_compute_ld<A, LOGN, L0, NP>(x, tw, q, qb, ninv, wlast);
    round_store<R, typename A::W, NP, LOGN>(x, sm);
    gs_rounds_smem_but_last_ld<A, LOGN, L0 + R::K, NP>(sm, tw, q, qb, ninv, wlast);
  }
}

template <int LOGN, int L0 = 0>
struct GsLast {
  static constexpr int value =
      (L0 + GsRound<LOGN, L0>::K >= LOGN) ? L0 : GsLast<LOGN, L0 + GsRound<LOGN, L0>::K>::value;
};
template <int LOGN>
struct GsLast<LOGN, LOGN> {
  static constexpr int value = LOGN;
};

}  // namespace secn
