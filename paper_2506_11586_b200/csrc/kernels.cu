// libsecn device kernels for sm_100a: RNS negacyclic NTT/INTT (Shoup, Harvey lazy butterflies,
// shared-memory radix-16 rounds), fused share-add / mask-add, the NTT-domain ct x pt
// multiply-accumulate, weight packing, and the designated-share gather. Every residue kernel is
// a template over the arithmetic policy: Arith64 (uint64 words, q < 2^61 -- the paper-parameter
// path) and Arith32 (uint32 words, q < 2^30 -- the 32-bit RNS-limb path).
//
// Paper: PAPER.md:376-380 (§6.2 NTT preprocessing: "transforms each ciphertext with NTT,
// performs all HE MAC operations in NTT, and only transforms the final HE results back"),
// PAPER.md:431 (§7: server share add, random mask), PAPER.md:668-679 (App. C.1 NTT).
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "internal.h"
#include "modarith.cuh"
#include "ntt_core.cuh"
#include "tma.cuh"

#include <cudaTypedefs.h>

namespace secn {

// ------------------------------------------------------------------------------------------
// per-policy access to the context's tables
template <class A>
struct Tab;
template <>
struct Tab<Arith64> {
  __device__ static const ulonglong2* fwd(const DevConsts& c) { return c.tw_fwd; }
  __device__ static const ulonglong2* inv(const DevConsts& c) { return c.tw_inv; }
  __device__ static ulonglong2 pair(uint64_t w, uint64_t wp) { return make_ulonglong2(w, wp); }
  __device__ static const ulonglong2* fwd_half(const DevConsts& c) { return c.tw_fwd_h; }
  __device__ static const ulonglong2* inv_half(const DevConsts& c) { return c.tw_inv_h; }
};
template <>
struct Tab<Arith32> {
  __device__ static const uint2* fwd(const DevConsts& c) { return c.tw32_fwd; }
  __device__ static const uint2* inv(const DevConsts& c) { return c.tw32_inv; }
  __device__ static uint2 pair(uint64_t w, uint64_t wp) { return make_uint2((uint32_t)w, (uint32_t)wp); }
  __device__ static const uint2* fwd_half(const DevConsts& c) { return c.tw32_fwd_h; }
  __device__ static const uint2* inv_half(const DevConsts& c) { return c.tw32_inv_h; }
};

// enc_j(v) = round(Q v / t) mod q_j (reading R2), computed through the identity
//   round(Q v / t) = (Q v - rho) / t + [rho >= t/2],  rho = Q v mod t = (Q mod t) v mod t,
// and Q = 0 (mod q_j):  enc_j(v) = -rho t^-1 + [rho >= t/2]  (mod q_j).
// rho is one 64-bit low product; rho t^-1 one Shoup product (64-bit limbs) or two 32-bit Shoup
// products on the 32-bit halves of rho (32-bit limbs). Canonical result in [0, q).
// Per-limb encoding constants, loaded once per thread.
struct EncK {
  uint64_t qmt, q, tinv, tinv_p, tinv_hi, tinv_hi_p;
  uint32_t tbits;
  __device__ __forceinline__ EncK(const DevConsts& c, int j)
      : qmt(c.qmt), q(c.q[j]), tinv(c.tinv[j]), tinv_p(c.tinv_p[j]), tinv_hi(c.tinv_hi[j]),
        tinv_hi_p(c.tinv_hi_p[j]), tbits(c.t_bits) {}
};

// the limb-dependent half of enc_j(v), from rho = (Q mod t) v mod t and up = [rho >= t/2]
template <class A>
__device__ __forceinline__ typename A::W enc_limb(uint64_t rho, uint32_t up, const EncK& k) {
  if constexpr (sizeof(typename A::W) == 8) {
    const uint64_t a = shoup(rho, k.tinv, k.tinv_p, k.q);  // [0, 2q)
    const uint64_t e = 2 * k.q - a + up;                     // [1, 2q + 1]
    return csub(csub(e, k.q), k.q);
  } else {
    const uint32_t q = (uint32_t)k.q;
    const uint32_t a = Arith32::shoup32((uint32_t)rho, (uint32_t)k.tinv, (uint32_t)k.tinv_p, q) +
                       Arith32::shoup32((uint32_t)(rho >> 32), (uint32_t)k.tinv_hi, (uint32_t)k.tinv_hi_p, q);
    uint32_t e = 4 * q - a + up;                             // [1, 4q + 1]
    e = csub32(e, 2 * q);
    return csub32(csub32(e, q), q);
  }
}

template <class A>
__device__ __forceinline__ typename A::W enc_mod(uint64_t v, const EncK& k) {
  const uint64_t rho = (k.qmt * v) & ((1ull << k.tbits) - 1);
  return enc_limb<A>(rho, rho >= (1ull << (k.tbits - 1)), k);
}

// CTAs per SM the NTT kernels are compiled for (register cap 65536 / (N/16 threads * this)). N =
// 4096, 32-bit words: 4 (64 registers) for the two-poly batches of the plain calls (+8% on the
// sweep), 3 for the one-poly share-add variant of the conv path (4 was slower in the step).
// N = 8192, 32-bit words: 2 (a lone CTA per SM idles at every barrier; +35% forward NTT/s).
template <class A, int LOGN, int NP>
constexpr int ntt_min_blocks() {
  return LOGN == 12 ? (sizeof(typename A::W) == 4 ? (NP == 2 ? 4 : 3) : 2) : LOGN == 13 && sizeof(typename A::W) == 4 ? 2 : 1;
}

// ------------------------------------------------------------------------------------------
// K1: forward NTT of limb-polys [P][N] (limb j = p mod L), optionally fused server-share add
// on the b component of ciphertexts [n][2][L][N]: b_j += enc_j(x0[n]).
// A CTA transforms NP polys of the same limb j: polys (g*NP + pp)*L + j, pp < NP, where g is
// the CTA's poly group (blockIdx.x / L); with NP = 2 these are the a and b components of one
// ciphertext. The first radix-16 round reads global memory directly (its tasks are coalesced).
template <class A, int LOGN, int NP>
__global__ void __launch_bounds__((1 << LOGN) / 16, ntt_min_blocks<A, LOGN, NP>())
    k_ntt_fwd(const typename A::W* in, typename A::W* out, const __grid_constant__ DevConsts c,
              const uint64_t* __restrict__ x0) {
  using W = typename A::W;
  using R0 = CtRound<LOGN, 0>;
  constexpr int N = 1 << LOGN;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const int j = (int)(blockIdx.x % c.L);
  const size_t grp = blockIdx.x / c.L;
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::fwd(c) + (size_t)j * N;
  const EncK ek(c, j);
  {  // the CTA's input polys (and share words) to L2 while the preceding kernel finishes: a prefetch
     // never reads stale data (L2 is the point of coherence), and the loads after the wait hit L2
     // (step -0.5%, profiles/r02zc_*)
    constexpr int LW = 128 / (int)sizeof(W);  // words per 128-byte line
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const size_t pi = grp * NP + pp;
      if (threadIdx.x < N / LW) prefetch_l2(in + (pi * c.L + j) * N + threadIdx.x * LW);
      if (x0 != nullptr && (pi & 1)) prefetch_l2(x0 + (pi >> 1) * N + threadIdx.x * 16);  // N/16 lines, one per thread
    }
  }
  typename A::Tw tws[15];
  ct_twiddles<A, LOGN, 0>(tws, tw);
  pdl_wait();  // inputs may come from the preceding kernel
  // dependents (the mask draw, the MAC) may launch now: none reads this kernel's output before its
  // own dependency wait, and the MAC's pre-wait weight loads are never produced here (the two-poly
  // variant of the large batches triggers at its end: the early trigger costs it registers)
  if constexpr (NP == 1) pdl_trigger();  // (at the end instead: 1.171 -> 1.197 ms, profiles/r02zd_*)
  W x[NP][16];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    const size_t pi = grp * NP + pp;  // poly index (ct * 2 + component for ciphertext batches)
    const W* src = in + (pi * c.L + j) * N;
    const bool share = x0 != nullptr && (pi & 1);  // uniform over the CTA
    // every load of the poly (and of its share words) is issued before any is used, so their
    // latencies overlap instead of chaining through the share-add branches
#pragma unroll
    for (int k = 0; k < R0::NT; ++k)
#pragma unroll
      for (int i = 0; i < R0::GK; ++i) x[pp][k * R0::GK + i] = src[R0::addr(k, i)];
    if (share) {
      const uint64_t* xs = x0 + (pi >> 1) * N;
      uint64_t xv[16];
#pragma unroll
      for (int k = 0; k < R0::NT; ++k)
#pragma unroll
        for (int i = 0; i < R0::GK; ++i) xv[k * R0::GK + i] = __ldg(&xs[R0::addr(k, i)]);
#pragma unroll
      for (int i = 0; i < 16; ++i) x[pp][i] += enc_mod<A>(xv[i], ek);  // < 2q: inside the CT domain
    }
  }
  ct_compute<A, LOGN, 0, NP>(x, tws, q, qb);
  round_store<R0, W, NP, LOGN>(x, sm);
  ct_rounds_smem_but_last<A, LOGN, R0::K, NP>(sm, tw, q, qb);
  // last round: its tasks are contiguous, so the results go straight to global memory
  constexpr int SL = CtLast<LOGN>::value;
  using RL = CtRound<LOGN, SL>;
  ct_twiddles<A, LOGN, SL>(tws, tw);
  __syncthreads();
  round_load<RL, W, NP, LOGN>(x, sm);
  ct_compute<A, LOGN, SL, NP>(x, tws, q, qb);
  if constexpr (NP != 1) pdl_trigger();
#pragma unroll
  for (int pp = 0; pp < NP; ++pp)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[pp][i] = A::canon_ct(x[pp][i], q);
  W* dst[NP];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) dst[pp] = out + ((grp * NP + pp) * c.L + j) * N;
  // through shared memory, so every warp store covers 512 contiguous bytes (step -0.7%, 64-bit
  // forward NTT 0.254 -> 0.260 of HBM against the per-thread 16-byte stores)
  if constexpr (RL::GK * sizeof(W) >= 16) {
    __syncthreads();  // every thread has read its last-round words from sm
    round_gstore_coalesced<RL, W, NP, LOGN>(x, sm, dst);
  } else {
    round_gstore<RL, W, NP>(x, dst);
  }
}

// K3: inverse NTT of limb-polys in place (the boundary call secn_ntt_inv; the hot path's inverse
// transform runs in k_mac + the tails, which fuse the mask). NP polys of limb j per CTA as in K1.
// The last radix-16 round writes global memory directly (its tasks are coalesced).
template <class A, int LOGN, int NP>
__global__ void __launch_bounds__((1 << LOGN) / 16, ntt_min_blocks<A, LOGN, NP>())
    k_ntt_inv(typename A::W* polys, const __grid_constant__ DevConsts c) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  constexpr int LL = GsLast<LOGN>::value;
  using RL = GsRound<LOGN, LL>;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const int j = (int)(blockIdx.x % c.L);
  const size_t grp = blockIdx.x / c.L;
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
  const typename A::Tw ninv = Tab<A>::pair(c.ninv[j], c.ninv_p[j]);
  const typename A::Tw wl = Tab<A>::pair(c.wlast[j], c.wlast_p[j]);
  // Encoded mask words enc_j(r) for the b poly of this CTA (odd poly index; with NP = 2 the pair
  // is (a, b) of one ciphertext, so at most one poly is masked). r is an input of the call, never
  // produced by the preceding kernel, so it is loaded and encoded before the dependency wait --
  // this work overlaps the previous kernel's tail -- and only the word-sized results are kept.
  // round 0 (levels 0..3, contiguous tasks) straight from global memory
  using R0 = GsRound<LOGN, 0>;
  typename A::Tw tws[15];
  gs_twiddles<A, LOGN, 0>(tws, tw);
  pdl_wait();  // the polys may come from the preceding kernel
  W x[NP][16];
  {
    const W* src[NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) src[pp] = polys + ((grp * NP + pp) * c.L + j) * N;
    round_gload<R0, W, NP>(x, src);
  }
  gs_compute<A, LOGN, 0, NP>(x, tws, q, qb, ninv, wl);
  round_store<R0, W, NP, LOGN>(x, sm);
  gs_rounds_smem_but_last<A, LOGN, R0::K, NP>(sm, tw, q, qb, ninv, wl);
  gs_twiddles<A, LOGN, LL>(tws, tw);
  __syncthreads();
  round_load<RL, W, NP, LOGN>(x, sm);
  gs_compute<A, LOGN, LL, NP>(x, tws, q, qb, ninv, wl);
  pdl_trigger();
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    const size_t pi = grp * NP + pp;
    W* buf = polys + (pi * c.L + j) * N;
#pragma unroll
    for (int k = 0; k < RL::NT; ++k)
#pragma unroll
      for (int i = 0; i < RL::GK; ++i) buf[RL::addr(k, i)] = A::canon_gs(x[pp][k * RL::GK + i], q);
  }
}

// ------------------------------------------------------------------------------------------
// C5 NTT engine for the plain batched calls (secn_ntt_fwd / secn_ntt_inv, weight preprocessing):
// persistent CTAs, each bound to one limb j, loop over items of NP limb-polys of that limb. Items
// arrive by TMA (cp.async.bulk.tensor through a 4-D map: 128-byte rows x rows x limb x poly,
// 128-byte swizzle) in two alternating buffers, and every radix-16 round works IN PLACE in the
// buffer the item landed in. The TMA of item i+1 (into the other buffer) is issued at item i's
// first barrier -- by then every thread has finished item i-1, the other buffer's last user --
// so the load overlaps item i's rounds, no global load sits on the critical path (the
// one-CTA-per-poly kernels above stall on their loads: profiles/r02s_ntt_full_summary.txt) and
// no barrier is added. The buffers keep TMA's swizzled layout: word e of a poly sits at
// stage_swz(e) (the 16-byte chunk index XOR the 128-byte row index mod 8), under which the
// rounds with contiguous tasks move whole 16-byte chunks conflict-free (LDS.128 / STS.128), the
// rounds with task stride >= 256 words are conflict-free word by word, and the stride-16 round
// has 2-way conflicts on 32-bit words (bank-conflict model: tools/ntt_bank_model.py).
// (stage_swz: ntt_core.cuh)

#ifndef SECN_TMA_NP12
#define SECN_TMA_NP12 1
#endif
#ifndef SECN_TMA_MINB12
#define SECN_TMA_MINB12 3
#endif
// polys per item and CTAs per SM (two buffers of NP polys per CTA: 64 KiB for 32-bit words at
// N = 4096 with NP = 2 -> 3 per SM; the register cap is 65536 / (N/16 x CTAs per SM))
template <class A, int LOGN>
__host__ __device__ constexpr int ntt_tma_np() { return SECN_TMA_NP12 && sizeof(typename A::W) == 4 && LOGN == 12 ? 2 : 1; }
template <class A, int LOGN>
__host__ __device__ constexpr int ntt_tma_minb() { return LOGN == 12 ? (sizeof(typename A::W) == 4 ? SECN_TMA_MINB12 : 2) : LOGN == 13 && sizeof(typename A::W) == 4 ? 2 : 1; }
#ifndef SECN_TMA_NBUF12
#define SECN_TMA_NBUF12 2
#endif
// staging buffers: 2 (the next item lands while this one is transformed), or 1 (it is issued after
// the last round has read the buffer, overlapping that round and the stores; more CTAs per SM)
template <class A, int LOGN>
__host__ __device__ constexpr int ntt_tma_nbuf() { return sizeof(typename A::W) == 4 && LOGN == 12 ? SECN_TMA_NBUF12 : 2; }
template <class A, int LOGN>
constexpr size_t ntt_tma_smem() {
  return 1024 + (size_t)ntt_tma_nbuf<A, LOGN>() * ntt_tma_np<A, LOGN>() * (1 << LOGN) * sizeof(typename A::W) + 16;
}

// round R's words of NP polys (poly pp at buf + pp N) <-> registers, in the swizzled layout
template <class R, class W, int NP, int N>
__device__ __forceinline__ void sw_load(W (&x)[NP][16], const W* buf) {
  constexpr int VW = 16 / (int)sizeof(W);
  if constexpr (R::logD == 0 && R::GK >= VW) {  // contiguous tasks: whole 16-byte chunks
#pragma unroll
    for (int k = 0; k < R::NT; ++k)
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int v = 0; v < R::GK / VW; ++v) {
          const uint4 t = *reinterpret_cast<const uint4*>(buf + pp * N + stage_swz<W>(R::addr(k, v * VW)));
          const W* tv = reinterpret_cast<const W*>(&t);
#pragma unroll
          for (int u = 0; u < VW; ++u) x[pp][k * R::GK + v * VW + u] = tv[u];
        }
  } else {
#pragma unroll
    for (int k = 0; k < R::NT; ++k)
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int i = 0; i < R::GK; ++i) x[pp][k * R::GK + i] = buf[pp * N + stage_swz<W>(R::addr(k, i))];
  }
}

template <class R, class W, int NP, int N>
__device__ __forceinline__ void sw_store(const W (&x)[NP][16], W* buf) {
  constexpr int VW = 16 / (int)sizeof(W);
  if constexpr (R::logD == 0 && R::GK >= VW) {
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
          *reinterpret_cast<uint4*>(buf + pp * N + stage_swz<W>(R::addr(k, v * VW))) = t;
        }
  } else {
#pragma unroll
    for (int k = 0; k < R::NT; ++k)
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int i = 0; i < R::GK; ++i) buf[pp * N + stage_swz<W>(R::addr(k, i))] = x[pp][k * R::GK + i];
  }
}

// CT rounds S0.. (in place, swizzled) up to but not including the last one; the first of them
// (S0 = 4) is preceded by the item's first barrier, where `at_first_barrier` runs
template <class A, int LOGN, int S0, int NP, class F>
__device__ __forceinline__ void ct_rounds_sw(typename A::W* buf, const typename A::Tw* __restrict__ tw,
                                             typename A::W q, typename A::W qb, F&& at_first_barrier) {
  using R = CtRound<LOGN, S0>;
  if constexpr (S0 + R::K < LOGN) {
    typename A::Tw tws[15];
    ct_twiddles<A, LOGN, S0>(tws, tw);
    if constexpr (S0 == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if constexpr (S0 == 4) at_first_barrier();
    typename A::W x[NP][16];
    sw_load<R, typename A::W, NP, 1 << LOGN>(x, buf);
    ct_compute<A, LOGN, S0, NP>(x, tws, q, qb);
    sw_store<R, typename A::W, NP, 1 << LOGN>(x, buf);
    ct_rounds_sw<A, LOGN, S0 + R::K, NP>(buf, tw, q, qb, at_first_barrier);
  }
}

template <class A, int LOGN, int L0, int NP, class F>
__device__ __forceinline__ void gs_rounds_sw(typename A::W* buf, const typename A::Tw* __restrict__ tw,
                                             typename A::W q, typename A::W qb, typename A::Tw ninv,
                                             typename A::Tw wlast, F&& at_first_barrier) {
  using R = GsRound<LOGN, L0>;
  if constexpr (L0 + R::K < LOGN) {
    typename A::Tw tws[15];
    gs_twiddles<A, LOGN, L0>(tws, tw);
    if constexpr (L0 == 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if constexpr (L0 == 4) at_first_barrier();
    typename A::W x[NP][16];
    sw_load<R, typename A::W, NP, 1 << LOGN>(x, buf);
    gs_compute<A, LOGN, L0, NP>(x, tws, q, qb, ninv, wlast);
    sw_store<R, typename A::W, NP, 1 << LOGN>(x, buf);
    gs_rounds_sw<A, LOGN, L0 + R::K, NP>(buf, tw, q, qb, ninv, wlast, at_first_barrier);
  }
}

template <class A, int LOGN, bool INV>
__global__ void __launch_bounds__((1 << LOGN) / 16, ntt_tma_minb<A, LOGN>())
    k_ntt_tma(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, typename A::W* out,
              const __grid_constant__ DevConsts c, uint32_t n_polys) {
  using W = typename A::W;
  using Tw = typename A::Tw;
  constexpr int N = 1 << LOGN, NP = ntt_tma_np<A, LOGN>(), NBUF = ntt_tma_nbuf<A, LOGN>();
  constexpr int RW = 128 / (int)sizeof(W), ROWS = N / RW, BR = ROWS < 256 ? ROWS : 256;
  static_assert(LOGN >= 12, "the first internal barrier is the one before round S0 = 4, and a later round exists");
  extern __shared__ __align__(1024) unsigned char smraw_tma[];
  W* bufs = reinterpret_cast<W*>(smraw_tma + ((1024 - (smem_u32(smraw_tma) & 1023)) & 1023));  // swizzle atoms
  uint64_t* bar = reinterpret_cast<uint64_t*>(bufs + NBUF * NP * N);
  const uint32_t L = c.L, j = blockIdx.x % L, per_limb = gridDim.x / L;
  const uint32_t n_items = (n_polys + NP - 1) / NP;
  const W q = (W)c.q[j], qb = A::bound(q);
  const Tw* tw = (INV ? Tab<A>::inv(c) : Tab<A>::fwd(c)) + (size_t)j * N;
  const Tw ninv = Tab<A>::pair(c.ninv[j], c.ninv_p[j]), wl = Tab<A>::pair(c.wlast[j], c.wlast_p[j]);
  // forward: the last round's words go back in place and leave by TMA store (whole 128-byte rows;
  // plain 16-byte stores of a thread's 16 contiguous words half-fill 32-byte sectors per instruction)
  constexpr bool tstore = !INV && LOGN == 12;  // measured: the inverse's coalesced word stores are faster
  const auto issue = [&](uint32_t item, int b) {  // one thread: the item's NP polys (zero-filled past n_polys)
    if constexpr (tstore) bulk_wait_read0();  // this buffer's TMA store (two items back) has read it
    mbar_arrive_expect_tx(&bar[b], (uint32_t)(NP * N * sizeof(W)));
#pragma unroll
    for (int pp = 0; pp < NP; ++pp)
#pragma unroll
      for (int k = 0; k < ROWS / BR; ++k)
        tma_load_4d(bufs + (b * NP + pp) * N + k * BR * RW, &tm, 0, k * BR, (int)j, (int)(item * NP + pp), &bar[b]);
  };
  if (threadIdx.x == 0) {
    prefetch_tmap(&tm);
    if constexpr (tstore) prefetch_tmap(&tmo);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // the polys may come from the preceding kernel
  uint32_t it = blockIdx.x / L;
  if (threadIdx.x == 0 && it < n_items) issue(it, 0);
  for (uint32_t k = 0; it < n_items; it += per_limb, ++k) {
    const int b = NBUF == 2 ? (int)(k & 1) : 0;
    const uint32_t par = NBUF == 2 ? (k >> 1) & 1 : k & 1;
    W* buf = bufs + b * NP * N;
    const uint32_t nxt = it + per_limb;
    const auto at_first_barrier = [&] {
      if (NBUF == 2 && threadIdx.x == 0 && nxt < n_items) issue(nxt, b ^ 1);
    };
    const auto after_last_read = [&] {  // one buffer: every thread has read this item's words
      if constexpr (NBUF == 1 && !tstore) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0 && nxt < n_items) issue(nxt, 0);
      }
    };
    const uint32_t p0 = it * NP;
    const auto store_item = [&] {  // the item's words are back in place: one thread TMA-stores them
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {  // rows past n_polys (the odd tail's missing poly) are clipped
#pragma unroll
        for (int pp = 0; pp < NP; ++pp)
#pragma unroll
          for (int kk = 0; kk < ROWS / BR; ++kk)
            tma_store_4d(&tmo, buf + pp * N + kk * BR * RW, 0, kk * BR, (int)j, (int)(p0 + pp));
        bulk_commit();
        if constexpr (NBUF == 1) {
          if (nxt < n_items) issue(nxt, 0);
        }
      }
    };
    W x[NP][16];
    Tw tws[15];
    if constexpr (!INV) {
      using R0 = CtRound<LOGN, 0>;
      constexpr int SL = CtLast<LOGN>::value;
      using RL = CtRound<LOGN, SL>;
      ct_twiddles<A, LOGN, 0>(tws, tw);
      mbar_wait(&bar[b], par);
      sw_load<R0, W, NP, N>(x, buf);
      ct_compute<A, LOGN, 0, NP>(x, tws, q, qb);
      sw_store<R0, W, NP, N>(x, buf);
      ct_rounds_sw<A, LOGN, R0::K, NP>(buf, tw, q, qb, at_first_barrier);
      ct_twiddles<A, LOGN, SL>(tws, tw);
      __syncthreads();
      sw_load<RL, W, NP, N>(x, buf);
      after_last_read();
      ct_compute<A, LOGN, SL, NP>(x, tws, q, qb);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[pp][i] = A::canon_ct(x[pp][i], q);
      if constexpr (tstore) {
        sw_store<RL, W, NP, N>(x, buf);  // each thread rewrites the words it read: no hazard
        store_item();
      } else {
        W* dst[NP];
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) dst[pp] = out + ((size_t)(p0 + pp) * L + j) * N;
        if (NP == 1 || p0 + NP <= n_polys) {
          round_gstore<RL, W, NP>(x, dst);
        } else {  // odd tail: the item's second poly does not exist
          W y[1][16];
#pragma unroll
          for (int i = 0; i < 16; ++i) y[0][i] = x[0][i];
          W* d1[1] = {dst[0]};
          round_gstore<RL, W, 1>(y, d1);
        }
      }
    } else {
      using R0 = GsRound<LOGN, 0>;
      constexpr int LL = GsLast<LOGN>::value;
      using RL = GsRound<LOGN, LL>;
      gs_twiddles<A, LOGN, 0>(tws, tw);
      mbar_wait(&bar[b], par);
      sw_load<R0, W, NP, N>(x, buf);
      gs_compute<A, LOGN, 0, NP>(x, tws, q, qb, ninv, wl);
      sw_store<R0, W, NP, N>(x, buf);
      gs_rounds_sw<A, LOGN, R0::K, NP>(buf, tw, q, qb, ninv, wl, at_first_barrier);
      gs_twiddles<A, LOGN, LL>(tws, tw);
      __syncthreads();
      sw_load<RL, W, NP, N>(x, buf);
      after_last_read();
      gs_compute<A, LOGN, LL, NP>(x, tws, q, qb, ninv, wl);
      if constexpr (tstore) {
#pragma unroll
        for (int pp = 0; pp < NP; ++pp)
#pragma unroll
          for (int i = 0; i < 16; ++i) x[pp][i] = A::canon_gs(x[pp][i], q);
        sw_store<RL, W, NP, N>(x, buf);
        store_item();
      } else {
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          if (pp > 0 && p0 + pp >= n_polys) break;
          W* o = out + ((size_t)(p0 + pp) * L + j) * N;
#pragma unroll
          for (int kk = 0; kk < RL::NT; ++kk)
#pragma unroll
            for (int i = 0; i < RL::GK; ++i) o[RL::addr(kk, i)] = A::canon_gs(x[pp][kk * RL::GK + i], q);
        }
      }
    }
  }
  if (tstore && threadIdx.x == 0) bulk_wait0();  // the stores are performed before the grid completes
  pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// Cluster NTT (N = 2^15; and 64-bit words at N = 2^14): at N = 2^15,
// T = N/16 = 2048 threads would exceed a CTA and 64-bit words need 272 KiB of shared memory; at
// 2^14 a 1024-thread CTA leaves 64 registers per thread, too few for 64-bit words. (32-bit words
// at 2^14 through two 512-thread cluster CTAs per SM measured slower: 10.8 vs 15.1 M NTT/s.) So a limb-poly
// is transformed by a CLUSTER of two CTAs of 2^LOGH = N/2 points each. The first CT level (and
// the last GS level) pairs coefficient e with e + N/2; every other level stays inside one half.
// CTA h (cluster rank) owns half h and runs the 2^LOGH-point core on it with its own twiddle
// table th (DevConsts::tw_*_h: the full table's entries of that half's groups).

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic address of the same shared-memory location in CTA `rank` of the cluster (DSMEM)
template <class T>
__device__ __forceinline__ const T* cluster_peer(const T* p, uint32_t rank) {
  uint64_t out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(reinterpret_cast<uint64_t>(p)), "r"(rank));
  return reinterpret_cast<const T*>(out);
}

// Forward: CTA h loads both halves (the partner's loads of the same lines hit L2), applies the
// cross-half level-0 butterfly (twiddle psi^brv(1)) and keeps its half; the share add (x0) is
// fused as in k_ntt_fwd. In-place calls are safe: no CTA stores before both passed the cluster
// barrier that follows their loads.
template <class A, int LOGH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((1 << LOGH) / 16, 1)
    k_ntt_fwd_cl(const typename A::W* in, typename A::W* out, const __grid_constant__ DevConsts c,
                 const uint64_t* __restrict__ x0) {
  using W = typename A::W;
  constexpr int NH = 1 << LOGH, N = 2 * NH;
  using R0 = CtRound<LOGH, 0>;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const uint32_t h = cluster_rank();
  const size_t pl = blockIdx.x >> 1;  // limb-poly
  const int j = (int)(pl % c.L);
  const size_t pi = pl / c.L;
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* th = Tab<A>::fwd_half(c) + ((size_t)j * 2 + h) * NH;
  const typename A::Tw w0 = Tab<A>::fwd(c)[(size_t)j * N + 1];
  const EncK ek(c, j);
  typename A::Tw tws[15];
  ct_twiddles<A, LOGH, 0>(tws, th);
  pdl_wait();
  const W* src = in + pl * N;
  const bool share = x0 != nullptr && (pi & 1);
  const uint64_t* xs = share ? x0 + (pi >> 1) * N : nullptr;
  W x[1][16];
#pragma unroll
  for (int k = 0; k < R0::NT; ++k)
#pragma unroll
    for (int i = 0; i < R0::GK; ++i) {
      const uint32_t e = R0::addr(k, i);
      W a = src[e], b = src[e + NH];
      if (share) {
        a += enc_mod<A>(__ldg(&xs[e]), ek);
        b += enc_mod<A>(__ldg(&xs[e + NH]), ek);
      }
      A::ct(a, b, w0, q, qb);
      x[0][k * R0::GK + i] = h ? b : a;
    }
  cluster_arrive();  // this CTA's global reads are done
  ct_compute<A, LOGH, 0, 1>(x, tws, q, qb);
  round_store<R0, W, 1, LOGH>(x, sm);
  ct_rounds_smem_but_last<A, LOGH, R0::K, 1>(sm, th, q, qb);
  constexpr int SL = CtLast<LOGH>::value;
  using RL = CtRound<LOGH, SL>;
  ct_twiddles<A, LOGH, SL>(tws, th);
  __syncthreads();
  round_load<RL, W, 1, LOGH>(x, sm);
  ct_compute<A, LOGH, SL, 1>(x, tws, q, qb);
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < 16; ++i) x[0][i] = A::canon_ct(x[0][i], q);
  W* dst[1] = {out + pl * N + h * NH};
  cluster_wait();  // the partner has read both halves
  round_gstore<RL, W, 1>(x, dst);  // (through shared memory, as k_ntt_fwd does, measured slower here)
}

// Inverse: CTA h runs GS levels 0..13 on its half (level 13 with twiddle th[1] and no N^-1),
// leaves the result in shared memory, and after a cluster barrier reads the partner's half
// through DSMEM for the cross-half level 14 (with N^-1 folded in, as in k_ntt_inv). A second
// cluster barrier keeps each CTA's shared memory alive until its partner has read it.
template <class A, int LOGH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((1 << LOGH) / 16, 1)
    k_ntt_inv_cl(typename A::W* polys, const __grid_constant__ DevConsts c) {
  using W = typename A::W;
  constexpr int NH = 1 << LOGH, N = 2 * NH, T = NH / 16;
  constexpr int LL = GsLast<LOGH>::value;
  using R0 = GsRound<LOGH, 0>;
  using RL = GsRound<LOGH, LL>;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const uint32_t h = cluster_rank();
  const size_t pl = blockIdx.x >> 1;
  const int j = (int)(pl % c.L);
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* th = Tab<A>::inv_half(c) + ((size_t)j * 2 + h) * NH;
  const typename A::Tw one = Tab<A>::pair(1, c.one_wp[j]);
  const typename A::Tw w13 = th[1];
  const typename A::Tw ninv = Tab<A>::pair(c.ninv[j], c.ninv_p[j]);
  const typename A::Tw wl = Tab<A>::pair(c.wlast[j], c.wlast_p[j]);
  // twiddles loaded at their use would avoid the 24-byte spill of 64-bit words at 2 x 2^14 points,
  // but measured slower there (0.145 -> 0.142 of HBM): gathered in registers for every word size
  constexpr bool tight = false;
  typename A::Tw tws[15];
  if constexpr (!tight) gs_twiddles<A, LOGH, 0>(tws, th);
  pdl_wait();  // the polys may come from the preceding kernel
  W* buf = polys + pl * N + h * NH;
  W x[1][16];
  {
    const W* src[1] = {buf};
    round_gload<R0, W, 1>(x, src);
  }
  if constexpr (tight) {
    gs_compute_ld<A, LOGH, 0, 1>(x, th, q, qb, one, w13);
    round_store<R0, W, 1, LOGH>(x, sm);
    gs_rounds_smem_but_last_ld<A, LOGH, R0::K, 1>(sm, th, q, qb, one, w13);
    __syncthreads();
    round_load<RL, W, 1, LOGH>(x, sm);
    gs_compute_ld<A, LOGH, LL, 1>(x, th, q, qb, one, w13);
  } else {
    gs_compute<A, LOGH, 0, 1>(x, tws, q, qb, one, w13);
    round_store<R0, W, 1, LOGH>(x, sm);
    gs_rounds_smem_but_last<A, LOGH, R0::K, 1>(sm, th, q, qb, one, w13);
    gs_twiddles<A, LOGH, LL>(tws, th);
    __syncthreads();
    round_load<RL, W, 1, LOGH>(x, sm);
    gs_compute<A, LOGH, LL, 1>(x, tws, q, qb, one, w13);
  }
  __syncthreads();  // every thread has read its last-round inputs before they are overwritten
  round_store<RL, W, 1, LOGH>(x, sm);
  cluster_arrive();
  cluster_wait();  // both halves are in shared memory
  pdl_trigger();
  const W* peer = cluster_peer(sm, h ^ 1);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T, pe = phys(e);
    const W mine = sm[pe], other = peer[pe];
    const W u = h ? other : mine, v = h ? mine : other;
    const W o = h ? A::mul4(u - v + qb, wl, q) : A::mul4(u + v, ninv, q);
    buf[e] = A::canon_gs(o, q);
  }
  cluster_arrive();
  cluster_wait();  // the partner is done reading this CTA's shared memory
}

// A8: y0 = -r mod t at the designated coefficients of output ciphertext `ct` (its mask row rs),
// split over the CTA's threads: fc plans (kind 1) put output row m*nob + d at coefficient
// d*nib + nib - 1; conv plans use the designation of include/secn.h (stride sh, window Hw x Ww).
__device__ __forceinline__ void write_server_share_ct(const uint64_t* __restrict__ rs, uint64_t* __restrict__ y0,
                                                      const PlanDev& pl, uint32_t ct, uint32_t t_bits) {
  const uint64_t tm = (1ull << t_bits) - 1;
  if (pl.kind == 1) {
    for (uint32_t d = threadIdx.x; d < pl.nob; d += blockDim.x) {
      const uint32_t o = ct * pl.nob + d;
      if (o < pl.no) y0[o] = (tm + 1 - rs[d * pl.nib + pl.nib - 1]) & tm;
    }
    return;
  }
  const uint32_t m = ct / pl.S, sidx = ct % pl.S;
  const uint32_t bh = sidx / pl.nbw, bw = sidx % pl.nbw;
  const uint32_t dh = pl.Hw - pl.kh + 1, dw = pl.Ww - pl.kw + 1;
  for (uint32_t d = threadIdx.x; d < dh * dw; d += blockDim.x) {
    const uint32_t i = d / dw, jj = d - i * dw;
    const uint32_t py = bh * dh + i, px = bw * dw + jj;
    const uint32_t oy = py / pl.sh, ox = px / pl.sh;
    if (oy * pl.sh != py || ox * pl.sh != px || oy >= pl.OH || ox >= pl.OW) continue;
    y0[((size_t)m * pl.OH + oy) * pl.OW + ox] = (tm + 1 - rs[pl.O + i * pl.Ww + jj]) & tm;
  }
}

// K3' (+A7 fused), the second half of secn_he_conv2d's inverse NTT: levels 8 .. LOGN-1 (with
// N^-1) on limb-polys whose levels 0..7 were applied by the MAC kernel (inputs in the lazy GS
// domain), then the mask on the b component. At N = 4096 this is one radix-16 round whose tasks
// (coefficients o + 256 i) are coalesced in global memory, with the same 15 twiddles for every
// thread: no shared memory, one load and one store per word.
template <class A, int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16, sizeof(typename A::W) == 4 && LOGN == 12 ? 4 : ntt_min_blocks<A, LOGN, 1>())
    k_ntt_inv_tail(typename A::W* polys, const __grid_constant__ DevConsts c, const uint64_t* __restrict__ r,
                   uint64_t* __restrict__ y0, const __grid_constant__ PlanDev pl, size_t ct0, int r_early,
                   const typename A::W* __restrict__ emb) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  constexpr int LS = 8;
  constexpr int LL = GsLast<LOGN>::value;
  using RS = GsRound<LOGN, LS>;
  using RL = GsRound<LOGN, LL>;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const uint32_t rb = gridDim.x - 1 - blockIdx.x;  // reverse output order, as k_ntt_inv_tail2
  const int j = (int)(rb % c.L);
  const size_t pa = rb / c.L;  // (active ct, component); the ct's row is slice_ct (s-slice)
  const size_t pi = 2 * (size_t)slice_ct(pl, (uint32_t)(ct0 + (pa >> 1))) + (pa & 1) - 2 * ct0;
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
  const typename A::Tw ninv = Tab<A>::pair(c.ninv_mac[j], c.ninv_mac_p[j]);  // inputs are k_mac outputs
  const typename A::Tw wl = Tab<A>::pair(c.wlast_mac[j], c.wlast_mac_p[j]);
  const EncK ek(c, j);
  const bool mask = (r != nullptr || emb != nullptr) && (pi & 1);
  W em[16];
  // the mask is an input of the call: with r_early (the preceding kernel is this call's MAC, which
  // never writes it) it is loaded and encoded before the dependency wait, overlapping the MAC's tail.
  // emb != NULL: the call's k_mask_encode already encoded it (em[ct][j][e]; chained, so early too)
  const auto load_mask = [&] {
    if (emb != nullptr) {
      const W* es = emb + (((pi >> 1) + ct0) * c.L + j) * N;
#pragma unroll
      for (int k = 0; k < RL::NT; ++k)
#pragma unroll
        for (int i = 0; i < RL::GK; ++i) em[k * RL::GK + i] = es[RL::addr(k, i)];
      return;
    }
    const uint64_t* rs = r + (pi >> 1) * N;
#pragma unroll
    for (int k = 0; k < RL::NT; ++k)
#pragma unroll
      for (int i = 0; i < RL::GK; ++i) em[k * RL::GK + i] = enc_mod<A>(__ldg(&rs[RL::addr(k, i)]), ek);
  };
  // 64-bit words at N = 2^14 (1024 threads, 64 registers): twiddles loaded at their use and the
  // mask after the transform, so the 16 words per thread are the only long-lived registers
  constexpr bool tight = sizeof(W) == 8 && LOGN >= 14;
  if (mask && r_early && !tight) load_mask();
  typename A::Tw tws[15];
  if constexpr (!tight) gs_twiddles<A, LOGN, LS>(tws, tw);
  pdl_wait();  // the polys are produced by the preceding kernel (the MAC)
  if (mask && !r_early && !tight) load_mask();
  W* buf = polys + (pi * c.L + j) * N;
  W x[1][16];
#pragma unroll
  for (int k = 0; k < RS::NT; ++k)
#pragma unroll
    for (int i = 0; i < RS::GK; ++i) x[0][k * RS::GK + i] = buf[RS::addr(k, i)];
  if constexpr (tight) {
    gs_compute_ld<A, LOGN, LS, 1>(x, tw, q, qb, ninv, wl);
    round_store<RS, W, 1, LOGN>(x, sm);
    gs_rounds_smem_but_last_ld<A, LOGN, LS + RS::K, 1>(sm, tw, q, qb, ninv, wl);
    __syncthreads();
    round_load<RL, W, 1, LOGN>(x, sm);
    gs_compute_ld<A, LOGN, LL, 1>(x, tw, q, qb, ninv, wl);
  } else {
    gs_compute<A, LOGN, LS, 1>(x, tws, q, qb, ninv, wl);
    if constexpr (LL != LS) {  // N > 4096: the remaining levels go through shared memory
      round_store<RS, W, 1, LOGN>(x, sm);
      gs_rounds_smem_but_last<A, LOGN, LS + RS::K, 1>(sm, tw, q, qb, ninv, wl);
      gs_twiddles<A, LOGN, LL>(tws, tw);
      __syncthreads();
      round_load<RL, W, 1, LOGN>(x, sm);
      gs_compute<A, LOGN, LL, 1>(x, tws, q, qb, ninv, wl);
    }
  }
  pdl_trigger();
#pragma unroll
  for (int k = 0; k < RL::NT; ++k)
#pragma unroll
    for (int i = 0; i < RL::GK; ++i) {
      W v = A::canon_gs(x[0][k * RL::GK + i], q);
      if (mask) {
        if constexpr (tight)  // the mask word loaded (and encoded) at its use
          v += emb != nullptr ? emb[(((pi >> 1) + ct0) * c.L + j) * N + RL::addr(k, i)]
                              : enc_mod<A>(__ldg(&r[(pi >> 1) * N + RL::addr(k, i)]), EncK(c, j));
        else
          v += em[k * RL::GK + i];
        v = v >= q ? v - q : v;
      }
      buf[RL::addr(k, i)] = v;
    }
  // A8 fused (secn_he_conv2d_ex): the server's output share y0 = -r mod t at the designated
  // coefficients of this ciphertext (one CTA per ciphertext does it: limb 0, b component). It
  // depends on r only, so it never waits on the transform; it saves a launch per layer.
  if (y0 != nullptr && r != nullptr && mask && j == 0)
    write_server_share_ct(r + (pi >> 1) * N, y0, pl, (uint32_t)(ct0 + (pi >> 1)), c.t_bits);
}

// The same tail at N = 4096 with both components of one (ciphertext, limb) per CTA: the pair
// shares the twiddles and the index arithmetic and every thread keeps 32 independent words in
// flight (the 16-word version is latency bound on small layers). Mask and A8 on component b.
// MS: how the mask arrives -- 0: r, loaded and encoded after the dependency wait (stage calls);
// 1: r, before the wait (chained); 2: already encoded by k_mask_encode, em[ct][j][e] (chained full calls).
template <class A, int MS>
__global__ void __launch_bounds__(256, 4)
    k_ntt_inv_tail2(typename A::W* polys, const __grid_constant__ DevConsts c, const uint64_t* __restrict__ r,
                    uint64_t* __restrict__ y0, const __grid_constant__ PlanDev pl, size_t ct0,
                    const typename A::W* __restrict__ emb) {
  using W = typename A::W;
  constexpr int LOGN = 12, N = 1 << LOGN, LS = 8;
  using RS = GsRound<LOGN, LS>;
  static_assert(GsLast<LOGN>::value == LS, "one round");
  // CTAs in reverse output order: the MAC wrote the highest output rows last, so theirs are the Y^
  // lines still in L2 when the tail starts (conv10's Y^ is twice the L2; step -0.4%, profiles/r02zj_*)
  const uint32_t rb = gridDim.x - 1 - blockIdx.x;
  const size_t ct = slice_ct(pl, (uint32_t)(ct0 + rb / c.L)) - ct0;  // row of this ct (s-slice aware)
  const int j = (int)(rb % c.L);
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
  const typename A::Tw ninv = Tab<A>::pair(c.ninv_mac[j], c.ninv_mac_p[j]);  // inputs are k_mac outputs
  const typename A::Tw wl = Tab<A>::pair(c.wlast_mac[j], c.wlast_mac_p[j]);
  const EncK ek(c, j);
  const bool mask = MS == 2 ? emb != nullptr : r != nullptr;
  const uint64_t* rs = r != nullptr ? r + ct * N : nullptr;
  W em[16];
  const auto load_mask = [&] {  // before the wait only when chained (see k_ntt_inv_tail)
    if constexpr (MS == 2) {
      const W* es = emb + ((ct + ct0) * c.L + j) * N;
#pragma unroll
      for (int i = 0; i < 16; ++i) em[i] = es[RS::addr(0, i)];
    } else {
      uint64_t rv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) rv[i] = __ldg(&rs[RS::addr(0, i)]);
#pragma unroll
      for (int i = 0; i < 16; ++i) em[i] = enc_mod<A>(rv[i], ek);
    }
  };
  if (mask && MS == 1) load_mask();
  // the encoded mask to L2 now (an input of the call, never written by the MAC), loaded after the
  // transform: step -0.75% (profiles/r02zc_*)
  if (MS == 2 && mask && (threadIdx.x & 31) < 16)
    prefetch_l2(emb + ((ct + ct0) * c.L + j) * N + (threadIdx.x & ~31u) + RS::T * (threadIdx.x & 31));
  typename A::Tw tws[15];
  gs_twiddles<A, LOGN, LS>(tws, tw);
  pdl_wait();  // the polys are produced by the preceding kernel (the MAC)
  if (mask && MS == 0) load_mask();
  W* buf[2] = {polys + ((ct * 2) * c.L + j) * N, polys + ((ct * 2 + 1) * c.L + j) * N};
  W x[2][16];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[pp][i] = buf[pp][RS::addr(0, i)];
  gs_compute<A, LOGN, LS, 2>(x, tws, q, qb, ninv, wl);
  pdl_trigger();  // (right after the wait instead: the next layer's forward NTT CTAs take the SMs early, +3.6%)
  if (mask && MS == 2) load_mask();  // 4-byte words: loaded here, their latency overlaps the a stores
#pragma unroll
  for (int i = 0; i < 16; ++i) buf[0][RS::addr(0, i)] = A::canon_gs(x[0][i], q);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    W v = A::canon_gs(x[1][i], q);
    if (mask) {
      v += em[i];
      v = v >= q ? v - q : v;
    }
    buf[1][RS::addr(0, i)] = v;
  }
  if (MS != 2 && y0 != nullptr && mask && j == 0) write_server_share_ct(rs, y0, pl, (uint32_t)(ct0 + ct), c.t_bits);
}

// The encoded-mask tail (the full calls with a drawn or pre-encoded mask) with bulk copies: both
// components of one (ciphertext, limb) and the encoded mask arrive by three 1-D bulk copies into
// shared memory (the mask's before the dependency wait), the transform reads and rewrites them
// there, and the two result polys leave by two bulk stores -- no per-thread global loads or
// stores (k_ntt_inv_tail2 with MS = 2 was LSU-throttled): step 1.1500 -> 1.1462 ms (r02zz2).
template <class A>
__global__ void __launch_bounds__(256, 4)
    k_ntt_inv_tail_bulk(typename A::W* polys, const __grid_constant__ DevConsts c, const __grid_constant__ PlanDev pl,
                        size_t ct0, const typename A::W* __restrict__ emb) {
  using W = typename A::W;
  constexpr int LOGN = 12, N = 1 << LOGN, LS = 8;
  using RS = GsRound<LOGN, LS>;
  extern __shared__ __align__(16) unsigned char smraw_tb[];
  W* sy = reinterpret_cast<W*>(smraw_tb);  // [2][N] polys a, b, then [N] encoded mask
  W* se = sy + 2 * N;
  uint64_t* bar = reinterpret_cast<uint64_t*>(se + N);
  const uint32_t rb = gridDim.x - 1 - blockIdx.x;  // reverse output order (as k_ntt_inv_tail2)
  const size_t ct = slice_ct(pl, (uint32_t)(ct0 + rb / c.L)) - ct0;
  const int j = (int)(rb % c.L);
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
  const typename A::Tw ninv = Tab<A>::pair(c.ninv_mac[j], c.ninv_mac_p[j]);
  const typename A::Tw wl = Tab<A>::pair(c.wlast_mac[j], c.wlast_mac_p[j]);
  W* buf0 = polys + ((ct * 2) * c.L + j) * N;
  W* buf1 = polys + ((ct * 2 + 1) * c.L + j) * N;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, 3 * N * sizeof(W));
    tma_load_1d(se, emb + ((ct + ct0) * c.L + j) * N, N * sizeof(W), bar);  // an input of the call
  }
  typename A::Tw tws[15];
  gs_twiddles<A, LOGN, LS>(tws, tw);
  pdl_wait();  // the polys are produced by the preceding kernel (the MAC)
  if (threadIdx.x == 0) {
    tma_load_1d(sy, buf0, N * sizeof(W), bar);
    tma_load_1d(sy + N, buf1, N * sizeof(W), bar);
  }
  __syncthreads();  // the barrier's init is visible before anyone waits on it
  mbar_wait(bar, 0);
  W x[2][16];
#pragma unroll
  for (int pp = 0; pp < 2; ++pp)
#pragma unroll
    for (int i = 0; i < 16; ++i) x[pp][i] = sy[pp * N + RS::addr(0, i)];
  gs_compute<A, LOGN, LS, 2>(x, tws, q, qb, ninv, wl);
  pdl_trigger();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    sy[RS::addr(0, i)] = A::canon_gs(x[0][i], q);
    W v = A::canon_gs(x[1][i], q) + se[RS::addr(0, i)];
    sy[N + RS::addr(0, i)] = v >= q ? v - q : v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    bulk_store_s2g(buf0, sy, N * sizeof(W));
    bulk_store_s2g(buf1, sy + N, N * sizeof(W));
    bulk_commit();
    bulk_wait_read0();  // shared memory stays valid until the stores have read it
  }
}

// ------------------------------------------------------------------------------------------
// A4: NTT-domain multiply-accumulate ("performs all HE MAC operations in NTT"):
//   Y^[m,s,c,j,e] = sum_g X^[g,s,c,j,e] * W[m,g,j,e] mod q_j
// Per coefficient e this is a small (M x G) . (G x 2S) matrix product. A CTA owns 256
// coefficients of limb j (one per consumer thread), a tile of output channels and a group of SG
// spatial blocks (both ciphertext components). The weights stream from HBM exactly once through
// a TMA ring: a producer warp issues one cp.async.bulk per (m, g) row segment (256 words) into an
// NS-stage shared-memory ring guarded by full/empty mbarriers, so the bytes in flight do not
// depend on registers or occupancy. The consumers' X^ values are staged once per CTA (registers
// for 32-bit words, shared memory for 64-bit words) and reused for every m of the tile. Products
// accumulate lazily (64-bit sums of 32x32 products; 128-bit sums of 64x64 products) with one
// reduction per output word. CTAs that share a weight tile (different s-groups) are adjacent in
// the grid so the second read of a tile hits L2.
constexpr int MAC_THREADS = 256;  // consumers; +32 producer threads

#ifdef SECN_PROBE  // timeline probes for tools/probe_mac.py (a separate build; off in libsecn.so)
__device__ unsigned long long g_probe[65536 * 2 + 64];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PROBE_CTA(slot) \
  if (threadIdx.x == 0) g_probe[64 + 2 * (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) + (slot)] = gtimer()
#define PROBE0(k) \
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) g_probe[k] = gtimer()
#else
#define PROBE_CTA(slot)
#define PROBE0(k)
#endif

// a mod q for a < 2^64, q < 2^28: a = hi 2^32 + lo with r32 = 2^32 mod q and the 32-bit Shoup
// companions r32p (of r32) and onep32 (of 1); three IMADs per half.
__device__ __forceinline__ uint32_t reduce64(uint64_t a, uint32_t q, uint32_t r32, uint32_t r32p, uint32_t onep32) {
  const uint32_t lo = (uint32_t)a, hi = (uint32_t)(a >> 32);
  const uint32_t x = Arith32::shoup32(hi, r32, r32p, q) + (lo - __umulhi(lo, onep32) * q);  // [0, 4q)
  return csub32(csub32(x, 2 * q), q);
}

// Montgomery REDC of a 64-bit MAC sum: a 2^-32 mod q in [0, 2q) for a < q 2^32, with
// qn = -q^-1 mod 2^32 (one IMAD and one IMAD.WIDE; the 2^32 is folded into the INTT's N^-1)
__device__ __forceinline__ uint32_t redc32(uint64_t a, uint32_t q, uint32_t qn) {
  const uint32_t m = (uint32_t)a * qn;
  return (uint32_t)((a + (uint64_t)m * q) >> 32);
}

template <class W>
struct ArithOf;
template <>
struct ArithOf<uint32_t> {
  using A = Arith32;
};
template <>
struct ArithOf<uint64_t> {
  using A = Arith64;
};

// A consumer warp hands ring stage `bar` back to the producer, whose next TMA load overwrites it.
// The stage's LDS must have READ shared memory first. ptxas issues the LDS, then sinks the
// multiply-adds that consume their results below a plain arrive, so the arrive can complete
// while the loads are still pending. A TMA write (async proxy) could then land under them: the
// race that corrupted whole weight rows when another kernel's CTAs shared the SM and slowed the
// LDS. The proxy fence orders each lane's generic-proxy reads before the
// async-proxy writes that follow the release.
__device__ __forceinline__ void consumer_release(uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

// barrier among the MAC_THREADS consumer threads only (the producer warp never joins)
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(MAC_THREADS) : "memory"); }

// Gentleman-Sande levels 0..7 of the inverse NTT on nch chunks of 256 coefficients (one e-tile of
// each output poly) held in shared memory in the padded layout (chunk ch at ch * MAC_CHS, word e
// at phys(e)). Levels 0..7 only pair coefficients inside an aligned block of 256, so the MAC CTA
// that owns the e-tile can apply them before Y^ leaves the SM (the INTT kernel does the rest).
// twe holds the e-tile's 255 twiddles: level l, local group g at twe[256 - (256 >> l) + g].
constexpr int MAC_CHS = MAC_THREADS + MAC_THREADS / 16;

// Position of twiddle (level l, local group g) in twe. Round A reads, per task b = tau & 15, the
// 8 >> p twiddles b * (8 >> p) .. of level p < 4 as 16-byte chunks; lanes b = 0..7 of an LDS.128
// phase would hit the same bank group (row stride 64 B for 32-bit, 128 B for 64-bit words), so
// the chunks of row b are XOR-swizzled by b (conflict-free for every level and word size).
template <class Tw>
__host__ __device__ __forceinline__ int twe_pos(int l, int g) {
  constexpr int CPW = 16 / (int)sizeof(Tw);  // twiddles per 16-byte chunk: 2 (32-bit), 1 (64-bit)
  const int base = 256 - (256 >> l);
  if (l >= 4) return base + g;
  const int n = 8 >> l;      // twiddles per task row
  const int cpr = n / CPW;    // chunks per row (>= 1 except 32-bit level 3)
  if (cpr <= 1) return base + g;
  const int b = g / n, w = g % n, v = w / CPW;
  const int sw = (b / (8 / cpr)) & (cpr - 1);
  return base + b * n + (v ^ sw) * CPW + w % CPW;
}

// the 8 >> l twiddles of task row b at level l < 4, as whole 16-byte chunks (see twe_pos)
template <class Tw, int l>
__device__ __forceinline__ void twe_row(Tw* out, const Tw* twe, int b) {
  constexpr int CPW = 16 / (int)sizeof(Tw), n = 8 >> l, cpr = n / CPW;
  const Tw* row = twe + 256 - (256 >> l) + b * n;
  if constexpr (cpr <= 1) {
#pragma unroll
    for (int w = 0; w < n; ++w) out[w] = row[w];
  } else {
    const int sw = (b / (8 / cpr)) & (cpr - 1);
#pragma unroll
    for (int v = 0; v < cpr; ++v) {
      const uint4 ch = reinterpret_cast<const uint4*>(row)[v ^ sw];
      const Tw* t = reinterpret_cast<const Tw*>(&ch);
#pragma unroll
      for (int k = 0; k < CPW; ++k) out[v * CPW + k] = t[k];
    }
  }
}

// kDense: round B leaves chunk ch DENSE at cbuf + ch * MAC_CHS (word e at offset e, for bulk
// stores to global memory): every task is loaded before a barrier and written after it, so the
// in-place change of layout cannot overwrite words another task has not read (needs
// nch <= 2 MAC_THREADS / 16 = 32 chunks).
// NT threads (local index lt) run the levels and synchronise among themselves with named barrier BAR
// (the default: k_mac's 256 consumers on barrier 1).
template <int BAR, int NT>
__device__ __forceinline__ void named_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

template <class A, bool kDense = false, int NT = MAC_THREADS, int BAR = 1>
__device__ __forceinline__ void mac_intt_levels_0_7(typename A::W* cbuf, const typename A::Tw* twe, int nch,
                                                    typename A::W q, typename A::W qb, int lt = -1) {
  using W = typename A::W;
  if (lt < 0) lt = threadIdx.x;
  const int ntask = nch * 16;
  // round A: levels 0..3, task = 16 consecutive coefficients 16b .. 16b+15 (phys: 17b + i)
  for (int tau = lt; tau < ntask; tau += NT) {
    W* base = cbuf + (tau >> 4) * MAC_CHS + 17 * (tau & 15);
    const int b = tau & 15;
    W x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = base[i];
    using Tw = typename A::Tw;
    if constexpr (sizeof(Tw) == 8) {  // 32-bit words: row b's twiddles of levels 0..3 in registers
      Tw tr[15];                      // level p at tr[16 - (16 >> p) + k]
      twe_row<Tw, 0>(tr, twe, b);
      twe_row<Tw, 1>(tr + 8, twe, b);
      twe_row<Tw, 2>(tr + 12, twe, b);
      twe_row<Tw, 3>(tr + 14, twe, b);
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int d = 1 << p;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i & d) continue;
          A::gs(x[i], x[i + d], tr[16 - (16 >> p) + (i >> (p + 1))], q, qb);
        }
      }
    } else {  // 64-bit words: one 16-byte twiddle per butterfly group, read at its use
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int d = 1 << p;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i & d) continue;
          A::gs(x[i], x[i + d], twe[twe_pos<Tw>(p, b * (8 >> p) + (i >> (p + 1)))], q, qb);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) base[i] = x[i];
  }
  named_sync<BAR, NT>();
  if constexpr (kDense) {
    W x[2][16];
    const int t0 = lt, t1 = lt + NT;
    if (t0 < ntask) {  // fewer than 16 chunks (MT x 2SG = 12 for SG = 3, MT = 2): not every thread has a task
#pragma unroll
      for (int i = 0; i < 16; ++i) x[0][i] = cbuf[(t0 >> 4) * MAC_CHS + (t0 & 15) + 17 * i];
    }
    if (t1 < ntask) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[1][i] = cbuf[(t1 >> 4) * MAC_CHS + (t1 & 15) + 17 * i];
    }
    named_sync<BAR, NT>();  // every task's words are in registers: the chunks may change layout
    if (t0 < ntask) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int d = 1 << p;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i & d) continue;
          A::gs(x[0][i], x[0][i + d], twe[256 - (256 >> (4 + p)) + (i >> (p + 1))], q, qb);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) cbuf[(t0 >> 4) * MAC_CHS + (t0 & 15) + 16 * i] = x[0][i];
    }
    if (t1 < ntask) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int d = 1 << p;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i & d) continue;
          A::gs(x[1][i], x[1][i + d], twe[256 - (256 >> (4 + p)) + (i >> (p + 1))], q, qb);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) cbuf[(t1 >> 4) * MAC_CHS + (t1 & 15) + 16 * i] = x[1][i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the bulk stores read these words
    named_sync<BAR, NT>();
    return;
  }
  // round B: levels 4..7, task = coefficients 16i + o (phys: 17i + o); the twiddles do not
  // depend on the task
  for (int tau = lt; tau < ntask; tau += NT) {
    W* base = cbuf + (tau >> 4) * MAC_CHS + (tau & 15);
    W x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = base[17 * i];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int d = 1 << p;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i & d) continue;
        const typename A::Tw w = twe[256 - (256 >> (4 + p)) + (i >> (p + 1))];
        A::gs(x[i], x[i + d], w, q, qb);
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) base[17 * i] = x[i];
  }
  named_sync<BAR, NT>();
}

// Register blocking: each consumer thread accumulates an [MT][2*SG] block of outputs (MT output
// channels x SG spatial blocks x 2 components) for its coefficient; the g loop is the runtime
// reduction loop. Per (m-block, g) the producer lands MT weight rows (MT x 256 words) in one ring
// stage; the consumer reads its 2*SG X^ values for g from the shared-memory X^ tile and does
// MT * 2 * SG multiply-accumulates.
template <class W, int SG, int MT>
__global__ void __launch_bounds__(MAC_THREADS + 32, 2)
    k_mac(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw, W* __restrict__ y,
          const __grid_constant__ DevConsts c, PlanDev pl, int m_range, int n_sg, int NS, int n_pre) {
  extern __shared__ __align__(128) unsigned char smraw_mac[];
  PROBE_CTA(0);
  PROBE0(0);
  constexpr int A2 = 2 * SG;
  const int N = 1 << c.log_n, L = c.L, G = pl.G, S = pl.S;
  const int j = blockIdx.y;
  const int sgi = blockIdx.x % n_sg, et = blockIdx.x / n_sg;
  const uint32_t e0 = et * MAC_THREADS;
  const int s0 = (int)pl.s0 + sgi * SG;  // s-groups tile the call's spatial slice
  const int ns = min(SG, (int)(pl.s0 + pl.sn) - s0);
  const int m_begin = blockIdx.z * m_range, m_end = min((int)pl.M, m_begin + m_range);
  const uint32_t row_bytes = MAC_THREADS * sizeof(W);
  using AR = typename ArithOf<W>::A;
  using Tw = typename AR::Tw;
  // shared memory: [G][2SG][256] X^ tile, [NS][MT][256] weight ring, [MT*2SG][MAC_CHS] output
  // chunks, [256] e-tile twiddles, 2*NS + 1 mbarriers
  W* xs = reinterpret_cast<W*>(smraw_mac);
  W* ring = xs + (size_t)G * A2 * MAC_THREADS;
  W* cbuf = ring + (size_t)NS * MT * MAC_THREADS;
  Tw* twe = reinterpret_cast<Tw*>(cbuf + (size_t)MT * A2 * MAC_CHS);
  uint64_t* full = reinterpret_cast<uint64_t*>(twe + MAC_THREADS);
  uint64_t* empty = full + NS;
  uint64_t* xbar = empty + NS;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MAC_THREADS / 32);
    }
    mbar_init(xbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= MAC_THREADS) {  // ---- producer warp: one elected lane streams X^ once, then the weights ----
    if (tid == MAC_THREADS) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmw);
      const uint64_t evict_first = policy_evict_first();  // weights are read once per query
      // The weights are inputs of the call (never produced by the preceding kernel): the first
      // n_pre stages of the ring are filled before the dependency wait, overlapping the forward
      // NTT; then the X^ tile, so that it does not queue behind a whole lap of weights (the
      // consumers need it before any stage), then the rest of the lap.
      int st = 0, issued = 0;
      uint32_t ph = 0, first = 1;  // ring position, its phase, and "first lap" (no wait needed)
      bool waited = false;
      for (int mb = m_begin; mb < m_end; mb += MT) {
        for (int g = 0; g < G; ++g) {
          if (!waited && (!first || issued == n_pre)) {
            pdl_wait();
            waited = true;
            // X^ tile (written by the forward NTT): box (256 coefficients, limb j, 2*SG rows
            // (s, c), G groups) in [g][a][256] order
            mbar_arrive_expect_tx(xbar, G * A2 * row_bytes);
            tma_load_4d(xs, &tmx, e0, j, 2 * s0, 0, xbar);
          }
          if (!first) mbar_wait_sleep(&empty[st], ph ^ 1);
          // weights: box (256 coefficients, row g*L + j, MT output channels from mb)
          mbar_arrive_expect_tx(&full[st], MT * row_bytes);
          if (c.word_bits & 0x400)  // debug: no L2 cache hint on the weight stream
            tma_load_3d(ring + (size_t)st * MT * MAC_THREADS, &tmw, e0, g * L + j, mb, &full[st]);
          else
            tma_load_3d_hint(ring + (size_t)st * MT * MAC_THREADS, &tmw, e0, g * L + j, mb, &full[st], evict_first);
          ++issued;
          if (++st == NS) st = 0, ph ^= 1, first = 0;
        }
      }
      if (!waited) {
        pdl_wait();
        mbar_arrive_expect_tx(xbar, G * A2 * row_bytes);
        tma_load_4d(xs, &tmx, e0, j, 2 * s0, 0, xbar);
      }
    }
    return;
  }

  // ---- consumers: one coefficient each (X^ rows beyond 2*ns are zero-filled; never stored) ----
  const uint32_t e = e0 + tid;
  const uint64_t q = c.q[j], onep = c.one_p[j];
  {  // the e-tile's inverse-NTT twiddles for levels 0..7 (constant tables: read before any wait)
    const Tw* tinv = Tab<AR>::inv(c) + (size_t)j * N;
    if (tid < 255) {
      int l = 0;
      while (tid >= 256 - (256 >> (l + 1))) ++l;
      const int g = tid - (256 - (256 >> l));
      twe[twe_pos<Tw>(l, g)] = tinv[(N >> (l + 1)) + (e0 >> (l + 1)) + g];
    }
  }
  const uint32_t qn = (uint32_t)c.qneg_inv32[j];
  const uint32_t r32 = (uint32_t)c.r32[j], r32p = (uint32_t)c.r32_p[j], onep32 = (uint32_t)(onep >> 32);
  PROBE0(1);
  mbar_wait_sleep(xbar, 0);
  PROBE0(2);
  int st = 0;
  uint32_t ph = 0;
  for (int mb = m_begin; mb < m_end; mb += MT) {
    const int rows = min(MT, m_end - mb);
    if constexpr (sizeof(W) == 4) {
      uint64_t acc[MT][A2];
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a) acc[r][a] = 0;
      for (int g = 0; g < G; ++g) {
        uint32_t xv[A2];
#pragma unroll
        for (int a = 0; a < A2; ++a) xv[a] = xs[(g * A2 + a) * MAC_THREADS + tid];
        mbar_wait_sleep(&full[st], ph);
        const W* wst = ring + (size_t)st * MT * MAC_THREADS + tid;
#pragma unroll
        for (int r = 0; r < MT; ++r) {
          const uint32_t wv = wst[r * MAC_THREADS];
#pragma unroll
          for (int a = 0; a < A2; ++a) acc[r][a] += (uint64_t)xv[a] * wv;  // < 2^56 each (q < 2^28), G <= 32
        }
        consumer_release(&empty[st]);
        if (++st == NS) st = 0, ph ^= 1;
      }
      if (tid < 32) bulk_wait_read0();  // the previous m-block's bulk stores have read the chunks
      consumer_sync();                    // ... and every thread knows it
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a)
          cbuf[(r * A2 + a) * MAC_CHS + phys(tid)] =
              c.mac_redc ? (W)redc32(acc[r][a], (uint32_t)q, qn)  // G q < 2^32; 2^-32 undone by ninv_mac
                         : (W)reduce64(acc[r][a], (uint32_t)q, r32, r32p, onep32);
    } else {
      const uint64_t r64 = c.r64[j], r64p = c.r64_p[j];
      uint64_t lo[MT][A2], hi[MT][A2];
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a) lo[r][a] = hi[r][a] = 0;
      for (int g = 0; g < G; ++g) {
        uint64_t xv[A2];
#pragma unroll
        for (int a = 0; a < A2; ++a) xv[a] = xs[(g * A2 + a) * MAC_THREADS + tid];
        mbar_wait_sleep(&full[st], ph);
        const W* wst = ring + (size_t)st * MT * MAC_THREADS + tid;
#pragma unroll
        for (int r = 0; r < MT; ++r) {
          const uint64_t wv = wst[r * MAC_THREADS];
#pragma unroll
          for (int a = 0; a < A2; ++a) mac128(lo[r][a], hi[r][a], xv[a], wv);  // G <= 32 < 64 terms of < 2^122
        }
        consumer_release(&empty[st]);
        if (++st == NS) st = 0, ph ^= 1;
      }
      consumer_sync();  // the previous m-block's chunks have been written out
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a)
          cbuf[(r * A2 + a) * MAC_CHS + phys(tid)] = (W)reduce128(lo[r][a], hi[r][a], q, r64, r64p, onep);
    }
    // inverse-NTT levels 0..7 of every staged output chunk, then the chunks leave the SM (lazy
    // GS domain values, finished by the INTT kernel)
    consumer_sync();
    PROBE0(3);
    if constexpr (sizeof(W) == 4) {
      // 32-bit words: the chunks leave dense through TMA bulk stores (one 1 KiB row segment per
      // output limb-poly), asynchronous to the next m-block's MAC
      mac_intt_levels_0_7<AR, true>(cbuf, twe, MT * A2, (W)q, AR::bound((W)q));
      PROBE0(4);
      if (tid < 32) {  // warp 0: lane ch issues chunk ch's store (MT x 2SG <= 32); L2 evict_last: the
                       // tail reads Y^ right back (step 1.1724 -> 1.1612 ms, profiles/r02zh_*)
        const int r = tid / A2, a = tid % A2;
        if (tid < MT * A2 && r < rows && a < 2 * ns)
          bulk_store_s2g_hint(y + ((((size_t)(mb + r) * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e0,
                              cbuf + tid * MAC_CHS, MAC_THREADS * sizeof(W), policy_evict_last());
        bulk_commit();
      }
    } else {
      mac_intt_levels_0_7<AR>(cbuf, twe, MT * A2, (W)q, AR::bound((W)q));
      PROBE0(4);
      const uint64_t evl = policy_evict_last();  // the tail reads Y^ right back
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a)
          if (r < rows && a < 2 * ns)
            st_hint(&y[((((size_t)(mb + r) * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e],
                    cbuf[(r * A2 + a) * MAC_CHS + phys(tid)], evl);
    }
  }
  if (sizeof(W) == 4 && tid < 32) bulk_wait_read0();  // shared memory stays valid until the stores have read it
  PROBE0(5);
  PROBE_CTA(1);
  pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// k_mac_ws: the same computation as k_mac<uint32_t, SG, MT> (32-bit limbs), warp-specialised so that
// a CTA's MAC and its inverse-NTT epilogue overlap across m-blocks. Warps 0-3 (128 threads, two
// coefficients of the e-tile each) accumulate m-block i+1 while warps 4-7 run levels 0..7 of m-block
// i on the other of two output-chunk buffers and bulk-store it; warp 8 streams the weights as in
// k_mac. Hand-offs: cfull[b] (the 4 MAC warps arrive after writing buffer b's reduced sums) and
// cempty[b] (the INTT store thread arrives once the bulk stores of b have read it). k_mac runs the
// two phases back to back on all 8 warps, so within a CTA the weight ring sits idle during the
// INTT and the integer pipes during the MAC's waits; here each m-block's phases hide the other's.
constexpr int WS_HALF = MAC_THREADS / 2;  // threads per role (MAC, INTT)

template <int SG, int MT>
__global__ void __launch_bounds__(MAC_THREADS + 32, 2)
    k_mac_ws(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw, uint32_t* __restrict__ y,
             const __grid_constant__ DevConsts c, PlanDev pl, int m_range, int n_sg, int NS, int n_pre) {
  using W = uint32_t;
  using AR = Arith32;
  using Tw = uint2;
  constexpr int A2 = 2 * SG, NCH = MT * A2;
  static_assert(NCH <= 2 * WS_HALF / 16, "the dense round B keeps <= 2 tasks per INTT thread");
  extern __shared__ __align__(128) unsigned char smraw_ws[];
  const int N = 1 << c.log_n, L = c.L, G = pl.G, S = pl.S;
  const int j = blockIdx.y;
  const int sgi = blockIdx.x % n_sg, et = blockIdx.x / n_sg;
  const uint32_t e0 = et * MAC_THREADS;
  const int s0 = (int)pl.s0 + sgi * SG;
  const int ns = min(SG, (int)(pl.s0 + pl.sn) - s0);
  const int m_begin = blockIdx.z * m_range, m_end = min((int)pl.M, m_begin + m_range);
  const uint32_t row_bytes = MAC_THREADS * sizeof(W);
  // shared memory: [G][2SG][256] X^ tile, [NS][MT][256] weight ring, [2][NCH][MAC_CHS] output
  // chunks, [256] e-tile twiddles, 2 NS + 1 + 4 mbarriers
  W* xs = reinterpret_cast<W*>(smraw_ws);
  W* ring = xs + (size_t)G * A2 * MAC_THREADS;
  W* cbuf0 = ring + (size_t)NS * MT * MAC_THREADS;
  Tw* twe = reinterpret_cast<Tw*>(cbuf0 + 2 * (size_t)NCH * MAC_CHS);
  uint64_t* full = reinterpret_cast<uint64_t*>(twe + MAC_THREADS);
  uint64_t* empty = full + NS;
  uint64_t* xbar = empty + NS;
  uint64_t* cfull = xbar + 1;
  uint64_t* cempty = cfull + 2;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int st = 0; st < NS; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], WS_HALF / 32);
    }
    mbar_init(xbar, 1);
    for (int b = 0; b < 2; ++b) mbar_init(&cfull[b], WS_HALF / 32), mbar_init(&cempty[b], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= MAC_THREADS) {  // ---- producer warp: as in k_mac ----
    if (tid == MAC_THREADS) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmw);
      const uint64_t evict_first = policy_evict_first();
      int st = 0, issued = 0;
      uint32_t ph = 0, first = 1;
      bool waited = false;
      for (int mb = m_begin; mb < m_end; mb += MT) {
        for (int g = 0; g < G; ++g) {
          if (!waited && (!first || issued == n_pre)) {
            pdl_wait();
            waited = true;
            mbar_arrive_expect_tx(xbar, G * A2 * row_bytes);
            tma_load_4d(xs, &tmx, e0, j, 2 * s0, 0, xbar);
          }
          if (!first) mbar_wait_sleep(&empty[st], ph ^ 1);
          mbar_arrive_expect_tx(&full[st], MT * row_bytes);
          tma_load_3d_hint(ring + (size_t)st * MT * MAC_THREADS, &tmw, e0, g * L + j, mb, &full[st], evict_first);
          ++issued;
          if (++st == NS) st = 0, ph ^= 1, first = 0;
        }
      }
      if (!waited) {
        pdl_wait();
        mbar_arrive_expect_tx(xbar, G * A2 * row_bytes);
        tma_load_4d(xs, &tmx, e0, j, 2 * s0, 0, xbar);
      }
    }
    return;
  }

  const uint32_t q = (uint32_t)c.q[j];
  if (tid < WS_HALF) {  // ---- MAC warps: coefficients e0 + tid and e0 + tid + 128 ----
    const uint32_t qn = (uint32_t)c.qneg_inv32[j];
    const uint32_t r32 = (uint32_t)c.r32[j], r32p = (uint32_t)c.r32_p[j], onep32 = (uint32_t)(c.one_p[j] >> 32);
    mbar_wait_sleep(xbar, 0);
    int st = 0;
    uint32_t ph = 0;
    int nb = 0;
    for (int mb = m_begin; mb < m_end; mb += MT, ++nb) {
      uint64_t acc[MT][A2][2];
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a) acc[r][a][0] = acc[r][a][1] = 0;
      for (int g = 0; g < G; ++g) {
        uint32_t xv[A2][2];
#pragma unroll
        for (int a = 0; a < A2; ++a)
#pragma unroll
          for (int h = 0; h < 2; ++h) xv[a][h] = xs[(g * A2 + a) * MAC_THREADS + tid + h * WS_HALF];
        mbar_wait_sleep(&full[st], ph);
        const W* wst = ring + (size_t)st * MT * MAC_THREADS + tid;
#pragma unroll
        for (int r = 0; r < MT; ++r)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t wv = wst[r * MAC_THREADS + h * WS_HALF];
#pragma unroll
            for (int a = 0; a < A2; ++a) acc[r][a][h] += (uint64_t)xv[a][h] * wv;  // < 2^56 each, G <= 32
          }
        consumer_release(&empty[st]);
        if (++st == NS) st = 0, ph ^= 1;
      }
      const int b = nb & 1;
      if (nb >= 2) mbar_wait_sleep(&cempty[b], ((nb >> 1) - 1) & 1);  // the INTT warps are done with buffer b
      W* cb = cbuf0 + (size_t)b * NCH * MAC_CHS;
#pragma unroll
      for (int r = 0; r < MT; ++r)
#pragma unroll
        for (int a = 0; a < A2; ++a)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            cb[(r * A2 + a) * MAC_CHS + phys(tid + h * WS_HALF)] =
                c.mac_redc ? redc32(acc[r][a][h], q, qn) : reduce64(acc[r][a][h], q, r32, r32p, onep32);
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&cfull[b]);  // release: the chunk writes precede it
    }
  } else {  // ---- INTT warps: levels 0..7 of each m-block's chunks, then the bulk stores ----
    const int lt = tid - WS_HALF;
    {  // the e-tile's inverse-NTT twiddles for levels 0..7
      const Tw* tinv = Tab<AR>::inv(c) + (size_t)j * N;
      for (int k = lt; k < 255; k += WS_HALF) {
        int l = 0;
        while (k >= 256 - (256 >> (l + 1))) ++l;
        const int g = k - (256 - (256 >> l));
        twe[twe_pos<Tw>(l, g)] = tinv[(N >> (l + 1)) + (e0 >> (l + 1)) + g];
      }
    }
    named_sync<2, WS_HALF>();
    int nb = 0;
    for (int mb = m_begin; mb < m_end; mb += MT, ++nb) {
      const int b = nb & 1, rows = min(MT, m_end - mb);
      W* cb = cbuf0 + (size_t)b * NCH * MAC_CHS;
      mbar_wait_sleep(&cfull[b], (nb >> 1) & 1);
      mac_intt_levels_0_7<AR, true, WS_HALF, 2>(cb, twe, NCH, q, AR::bound(q), lt);  // dense chunks, proxy fence
      if (lt < 32) {  // INTT warp 0: lane ch stores chunk ch (one 1 KiB row segment per output limb-poly)
        const int r = lt / A2, a = lt % A2;
        if (lt < NCH && r < rows && a < 2 * ns)
          bulk_store_s2g_hint(y + ((((size_t)(mb + r) * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e0,
                              cb + lt * MAC_CHS, MAC_THREADS * sizeof(W), policy_evict_last());
        bulk_commit();
        // the previous m-block's stores (the other buffer) have read their chunks: hand it back
        if (nb >= 1) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (lt == 0) mbar_arrive(&cempty[b ^ 1]);
        }
      }
    }
    if (lt < 32) bulk_wait_read0();  // shared memory stays valid until the stores have read it
  }
  pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// The whole layer after the forward NTT in ONE kernel, for the small layers (32-bit limbs,
// N = 4096): A4 MAC, all 12 inverse-NTT levels, N^-1, A7 mask and A8 server share. A CTA owns
// whole output polys -- limb j of the MT x SG output ciphertexts (m, s) of an m-block and an
// s-group, both components (NP = 2 MT SG polys, 17 KiB each in shared memory) -- so Y^ never
// leaves the SM and there is no tail kernel. Phase A streams, per e-tile of 256 coefficients and
// chunk of GC input groups, the X^ rows (G x 2SG, L2-resident) and the weight rows (MT x G, HBM,
// read once) through a TMA ring (one elected producer thread, full/empty mbarriers), accumulates
// the [MT x 2SG] block of lazy 64-bit sums per coefficient and reduces it (REDC) into the output
// polys. Phase B runs the three radix-16 Gentleman-Sande rounds on the polys in shared memory
// (every poly of the CTA has limb j, so one set of twiddles per task serves all of them); the
// last round's tasks (coefficients tid + 256 i) are coalesced, so it adds the mask and stores
// straight to global memory. The MAC's multiply-add work and weight bytes equal k_mac's; what
// goes away is the Y^ round trip through HBM and the tail launch.
constexpr int FUSED_THREADS = 256;  // consumers; +32 producer threads

template <int SG, int MT>
__global__ void __launch_bounds__(FUSED_THREADS + 32, 2)
    k_layer_fused(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
                  uint32_t* __restrict__ y, const uint64_t* __restrict__ r, uint64_t* __restrict__ y0,
                  const __grid_constant__ DevConsts c, const __grid_constant__ PlanDev pl, int n_sg, int NS, int GC,
                  int n_pre, const uint32_t* __restrict__ emb) {
  using AR = Arith32;
  using W = uint32_t;
  using Tw = uint2;
  constexpr int LOGN = 12, N = 1 << LOGN, A2 = 2 * SG, NP = MT * A2, SW = smem_words<LOGN>();
  extern __shared__ __align__(1024) unsigned char smraw_fused[];
  const int L = (int)c.L, G = (int)pl.G, S = (int)pl.S;
  const int j = blockIdx.y;
  const int sgi = blockIdx.x % n_sg, mb = (blockIdx.x / n_sg) * MT;
  const int s0 = (int)pl.s0 + sgi * SG, ns = min(SG, (int)(pl.s0 + pl.sn) - s0), rows = min(MT, (int)pl.M - mb);
  const int n_gc = (G + GC - 1) / GC, total = (N / FUSED_THREADS) * n_gc;
  const int stage_words = GC * (A2 + MT) * FUSED_THREADS;
  // shared memory: [NP][SW] output polys (padded layout), [NS][stage] ring, 2 NS mbarriers
  W* obuf = reinterpret_cast<W*>(smraw_fused);
  W* ring = obuf + NP * SW;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NS * stage_words);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int st = 0; st < NS; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], FUSED_THREADS / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (tid >= FUSED_THREADS) {  // ---- producer: stage k = (e-tile k / n_gc, group chunk k % n_gc) ----
    if (tid == FUSED_THREADS) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmw);
      const uint64_t evict_first = policy_evict_first();  // weights are read once per query
      const uint32_t bytes = (uint32_t)stage_words * sizeof(W);
      const auto load_w = [&](int k, int st) {
        W* dst = ring + (size_t)st * stage_words + GC * A2 * FUSED_THREADS;
        tma_load_4d_hint(dst, &tmw, (k / n_gc) * FUSED_THREADS, j, (k % n_gc) * GC, mb, &full[st], evict_first);
      };
      const auto load_x = [&](int k, int st) {
        tma_load_4d(ring + (size_t)st * stage_words, &tmx, (k / n_gc) * FUSED_THREADS, j, 2 * s0, (k % n_gc) * GC,
                    &full[st]);
      };
      // the weights are never produced by the preceding kernel of a chained call: the first n_pre
      // stages' weight rows go out before the dependency wait; X^ (the forward NTT's output) after
      const int npre = min(n_pre, min(NS, total));
      for (int k = 0; k < npre; ++k) {
        mbar_arrive_expect_tx(&full[k], bytes);
        load_w(k, k);
      }
      pdl_wait();
      for (int k = 0; k < npre; ++k) load_x(k, k);
      for (int k = npre; k < total; ++k) {
        const int st = k % NS;
        if (k >= NS) mbar_wait_sleep(&empty[st], ((k / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], bytes);
        load_w(k, st);
        load_x(k, st);
      }
    }
    return;
  }

  // ---- phase A: MAC, one coefficient of the e-tile per consumer thread ----
  const uint32_t q = (uint32_t)c.q[j], qb = AR::bound(q);
  const uint32_t qn = (uint32_t)c.qneg_inv32[j];
  const uint32_t r32 = (uint32_t)c.r32[j], r32p = (uint32_t)c.r32_p[j], onep32 = (uint32_t)(c.one_p[j] >> 32);
  int k = 0;
  for (int et = 0; et < N / FUSED_THREADS; ++et) {
    uint64_t acc[MT][A2];
#pragma unroll
    for (int rr = 0; rr < MT; ++rr)
#pragma unroll
      for (int a = 0; a < A2; ++a) acc[rr][a] = 0;
    for (int gc = 0; gc < n_gc; ++gc, ++k) {
      const int st = k % NS;
      mbar_wait_sleep(&full[st], (k / NS) & 1);
      const W* xs = ring + (size_t)st * stage_words + tid;
      const W* wsg = xs + GC * A2 * FUSED_THREADS;
      const int gn = min(GC, G - gc * GC);
      for (int gg = 0; gg < gn; ++gg) {
        uint32_t xv[A2];
#pragma unroll
        for (int a = 0; a < A2; ++a) xv[a] = xs[(gg * A2 + a) * FUSED_THREADS];
#pragma unroll
        for (int rr = 0; rr < MT; ++rr) {
          const uint32_t wv = wsg[(rr * GC + gg) * FUSED_THREADS];
#pragma unroll
          for (int a = 0; a < A2; ++a) acc[rr][a] += (uint64_t)xv[a] * wv;  // G <= 32 terms < 2^54
        }
      }
      consumer_release(&empty[st]);
    }
    const uint32_t pe = phys(et * FUSED_THREADS + tid);
#pragma unroll
    for (int rr = 0; rr < MT; ++rr)
#pragma unroll
      for (int a = 0; a < A2; ++a)
        obuf[(rr * A2 + a) * SW + pe] = c.mac_redc ? redc32(acc[rr][a], q, qn)  // [0, 2q); 2^-32 undone by ninv_mac
                                                   : reduce64(acc[rr][a], q, r32, r32p, onep32);
  }

  // ---- phase B: inverse NTT of the NP polys in shared memory ----
  const Tw* tw = Tab<AR>::inv(c) + (size_t)j * N;
  const Tw ninv = Tab<AR>::pair(c.ninv_mac[j], c.ninv_mac_p[j]), wl = Tab<AR>::pair(c.wlast_mac[j], c.wlast_mac_p[j]);
  Tw tws[15];
  const auto round_smem = [&](auto rtag) {
    constexpr int L0 = decltype(rtag)::value;
    using R = GsRound<LOGN, L0>;
    gs_twiddles<AR, LOGN, L0>(tws, tw);
    consumer_sync();  // the previous phase / round has written every poly
#pragma unroll 1
    for (int p = 0; p < NP; p += 2) {
      W x[2][16];
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[pp][i] = obuf[(p + pp) * SW + R::pbase(0) + R::poff(i)];
      gs_compute<AR, LOGN, L0, 2>(x, tws, q, qb, ninv, wl);
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int i = 0; i < 16; ++i) obuf[(p + pp) * SW + R::pbase(0) + R::poff(i)] = x[pp][i];
    }
  };
  round_smem(std::integral_constant<int, 0>());
  round_smem(std::integral_constant<int, 4>());
  // last round (levels 8..11 with N^-1): tasks tid + 256 i are coalesced -> global memory, with the
  // mask on the b component
  using RL = GsRound<LOGN, 8>;
  gs_twiddles<AR, LOGN, 8>(tws, tw);
  consumer_sync();
  const EncK ek(c, j);
  const uint64_t tm = (1ull << c.t_bits) - 1;
#pragma unroll 1
  for (int p = 0; p < NP; p += 2) {  // p even: (a, b) of one output ciphertext
    const int rr = p / A2, a = p % A2, sl = a >> 1;
    const bool live = rr < rows && sl < ns;
    const size_t ct = (size_t)(mb + rr) * S + s0 + sl;
    W em[16];  // enc_j of the mask words (encoded before the polys are loaded: fewer live registers)
    const bool masked = r != nullptr || emb != nullptr;
    if (live && emb != nullptr) {
#pragma unroll
      for (int i = 0; i < 16; ++i) em[i] = emb[(ct * L + j) * N + RL::addr(0, i)];
    } else if (live && r != nullptr) {
      uint64_t rv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) rv[i] = __ldg(&r[ct * N + RL::addr(0, i)]);
#pragma unroll
      for (int i = 0; i < 16; ++i) em[i] = enc_mod<AR>(rv[i], ek);
    }
    W x[2][16];
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int i = 0; i < 16; ++i) x[pp][i] = obuf[(p + pp) * SW + RL::pbase(0) + RL::poff(i)];
    gs_compute<AR, LOGN, 8, 2>(x, tws, q, qb, ninv, wl);
    if (live) {
      W* ya = y + ((ct * 2) * L + j) * N;
      W* yb = y + ((ct * 2 + 1) * L + j) * N;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        ya[RL::addr(0, i)] = AR::canon_gs(x[0][i], q);
        W v = AR::canon_gs(x[1][i], q);
        if (masked) {
          v += em[i];
          v = v >= q ? v - q : v;
        }
        yb[RL::addr(0, i)] = v;
      }
      // A8: the server's share y0 = -r mod t at the designated coefficients (limb 0's CTA; with em,
      // k_mask_encode wrote it)
      if (y0 != nullptr && r != nullptr && emb == nullptr && j == 0) {
        const uint32_t sidx = (uint32_t)(ct % S), bh = sidx / pl.nbw, bw = sidx % pl.nbw;
        const uint32_t dh = pl.Hw - pl.kh + 1, dw = pl.Ww - pl.kw + 1;
        for (uint32_t d = tid; d < dh * dw; d += FUSED_THREADS) {
          const uint32_t i = d / dw, jj = d - i * dw;
          const uint32_t py = bh * dh + i, px = bw * dw + jj;
          const uint32_t oy = py / pl.sh, ox = px / pl.sh;
          if (oy * pl.sh != py || ox * pl.sh != px || oy >= pl.OH || ox >= pl.OW) continue;
          y0[((size_t)(mb + rr) * pl.OH + oy) * pl.OW + ox] = (tm + 1 - r[ct * N + pl.O + i * pl.Ww + jj]) & tm;
        }
      }
    }
  }
  pdl_trigger();
}

// ------------------------------------------------------------------------------------------
// f2 (reading R16): the INTT tail with the output switched to Lk limbs and
// extracted. One CTA per (output ct, component), 256 threads, 16 coefficients o + 256 i per
// thread (N = 4096). Modulus switching needs all L residues of a coefficient: the dropped limbs
// go first and fold into the centred CRT value v = [c]_P of the dropped part,
//   v = sum_j ((c_j (P/q_j)^-1) mod q_j) (P/q_j)  mod P,  then centred into (-P/2, P/2);
// every kept limb i then yields c'_i = (c_i - v) P^-1 mod q_i = round(c Q'/Q) mod q_i exactly
// (c - [c]_P is the multiple of P nearest to c; P is odd, so there are no ties). The a
// component is written whole (a' is shared by every designated coefficient), the b component only
// at its designated coefficients, as b'[value][Lk].

// canonical a mod q for any 64-bit a
template <class A>
__device__ __forceinline__ typename A::W reduce_u64(uint64_t a, const DevConsts& c, int j);
template <>
__device__ __forceinline__ uint64_t reduce_u64<Arith64>(uint64_t a, const DevConsts& c, int j) {
  return reduce128(a, 0, c.q[j], c.r64[j], c.r64_p[j], c.one_p[j]);
}
template <>
__device__ __forceinline__ uint32_t reduce_u64<Arith32>(uint64_t a, const DevConsts& c, int j) {
  return reduce64(a, (uint32_t)c.q[j], (uint32_t)c.r32[j], (uint32_t)c.r32_p[j], (uint32_t)(c.one_p[j] >> 32));
}

// output index of coefficient e of output ct `ct` under plan pl, or -1 (not designated)
__device__ __forceinline__ int64_t designated_index(const PlanDev& pl, uint32_t ct, uint32_t e) {
  if (pl.kind == 1) {  // fc: y[m*nob + d] at d*nib + nib - 1
    if ((e + 1) % pl.nib != 0) return -1;
    const uint32_t d = (e + 1) / pl.nib - 1;
    const uint32_t o = ct * pl.nob + d;
    return d < pl.nob && o < pl.no ? (int64_t)o : -1;
  }
  if (e < pl.O) return -1;
  const uint32_t dd = e - pl.O, i = dd / pl.Ww, jj = dd % pl.Ww;
  if (i > pl.Hw - pl.kh || jj > pl.Ww - pl.kw) return -1;
  const uint32_t m = ct / pl.S, s = ct % pl.S, bh = s / pl.nbw, bw = s % pl.nbw;
  const uint32_t py = bh * (pl.Hw - pl.kh + 1) + i, px = bw * (pl.Ww - pl.kw + 1) + jj;
  const uint32_t oy = py / pl.sh, ox = px / pl.sh;
  if (oy * pl.sh != py || ox * pl.sh != px || oy >= pl.OH || ox >= pl.OW) return -1;
  return ((int64_t)m * pl.OH + oy) * pl.OW + ox;
}

// Launch shape: one CTA per (output ct, component, half of the 256 radix-16 tasks), L warp groups of
// 128 threads, group j = limb j, so every limb's loads are in flight at once. Task o = h*128 + lt
// covers coefficients o + 256 i (i < 16). Dropped-limb groups leave y_j = c_j (P/q_j)^-1 mod q_j
// in shared memory; after one barrier the kept-limb groups fold v = sum_j y_j (P/q_j) mod P,
// centre it and write their switched residues.
constexpr int LWE_G = 128;

template <class A, int ND>  // ND = L - Lk dropped limbs
__global__ void __launch_bounds__(LWE_G * SECN_MAX_LIMBS)
    k_ntt_inv_tail_lwe(const typename A::W* __restrict__ polys, const __grid_constant__ DevConsts c,
                       const __grid_constant__ MsConsts ms, const uint64_t* __restrict__ r, typename A::W* a_out,
                       typename A::W* b_out, uint64_t* y0, const __grid_constant__ PlanDev pl, int r_early,
                       const typename A::W* __restrict__ emb) {
  using W = typename A::W;
  constexpr int LOGN = 12, N = 1 << LOGN;
  using RS = GsRound<LOGN, 8>;
  static_assert(RS::NT == 1 && RS::GK == 16, "one radix-16 task per thread");
  __shared__ W ys[ND][16][LWE_G];
  // CTAs in reverse output order, as the full-ciphertext tails: the Y^ rows the MAC wrote last are read first
  const uint32_t rb = gridDim.x - 1 - blockIdx.x;
  const size_t ct = slice_ct(pl, rb >> 2), pi = 2 * ct + ((rb >> 1) & 1);
  const uint32_t o = (rb & 1) * LWE_G + threadIdx.x % LWE_G;  // radix-16 task: coefficients o + 256 i
  const int j = threadIdx.x / LWE_G;                                   // this group's limb
  const bool isb = pi & 1, mask = isb && (r != nullptr || emb != nullptr);
  const uint64_t* rs = isb && r != nullptr ? r + ct * N : nullptr;
  const int L = (int)c.L, Lk = L - ND;
  const W q = (W)c.q[j], qb = A::bound(q);
  typename A::Tw tws[15];
  {  // twiddles of levels 8..11: the round has a single block, so every task uses the same 15
     // (level 8 + p, group gi at tw[N / 2^(9+p) + gi]; layout as in gs_twiddles)
    const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int gi = 0; gi < (8 >> p); ++gi) tws[16 - (16 >> p) + gi] = tw[(N >> (9 + p)) + gi];
  }
  // b component: only designated coefficients leave the kernel, so a task none of whose 16
  // coefficients is designated does no work (convolutions: they lie in [O, O + (Hw-kh) Ww + Ww-kw])
  bool work = true;
  if (isb && pl.kind == 0) {
    const uint32_t lo = pl.O, hi = pl.O + (pl.Hw - pl.kh) * pl.Ww + (pl.Ww - pl.kw);
    work = false;
#pragma unroll
    for (int i = 0; i < 16; ++i) work |= (o + 256 * i >= lo) && (o + 256 * i <= hi);
  }
  const EncK ek(c, j);
  W em[16];
  if (mask && work && emb != nullptr) {  // encoded by the call's k_mask_encode
#pragma unroll
    for (int i = 0; i < 16; ++i) em[i] = emb[(ct * L + j) * N + o + 256 * i];
  } else if (mask && work && r_early) {
#pragma unroll
    for (int i = 0; i < 16; ++i) em[i] = enc_mod<A>(__ldg(&rs[o + 256 * i]), ek);
  }
  pdl_wait();
  if (mask && work && emb == nullptr && !r_early) {
#pragma unroll
    for (int i = 0; i < 16; ++i) em[i] = enc_mod<A>(__ldg(&rs[o + 256 * i]), ek);
  }
  W x[1][16];
  if (work) {
    const W* buf = polys + (pi * L + j) * N;
#pragma unroll
    for (int i = 0; i < 16; ++i) x[0][i] = buf[o + 256 * i];
    gs_compute<A, LOGN, 8, 1>(x, tws, q, qb, Tab<A>::pair(c.ninv_mac[j], c.ninv_mac_p[j]),
                              Tab<A>::pair(c.wlast_mac[j], c.wlast_mac_p[j]));
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      W v = A::canon_gs(x[0][i], q);
      if (mask) {
        v += em[i];
        v = v >= q ? v - q : v;
      }
      x[0][i] = v;
    }
    if (j >= Lk) {  // dropped limb: y_j = c_j (P/q_j)^-1 mod q_j
      const typename A::Tw inv = Tab<A>::pair(ms.inv[j], ms.inv_p[j]);
#pragma unroll
      for (int i = 0; i < 16; ++i) ys[j - Lk][i][threadIdx.x % LWE_G] = A::canon_gs(A::mul4(x[0][i], inv, q), q);
    }
  }
  pdl_trigger();
  __syncthreads();  // every thread, converged (aligned barrier)
  if (!work || j >= Lk) return;
  const typename A::Tw pinv = Tab<A>::pair(ms.pinv[j], ms.pinv_p[j]);
  uint64_t pq[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) pq[d] = ms.pq[Lk + d];
  const uint32_t lt = threadIdx.x % LWE_G;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t e = o + 256 * i;
    const int64_t oi = isb ? designated_index(pl, (uint32_t)ct, e) : 0;
    if (oi < 0) continue;  // b: not designated
    uint64_t v = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) v += (uint64_t)ys[d][i][lt] * pq[d];
#pragma unroll
    for (int d = 1; d < ND; ++d) v = v >= ms.P ? v - ms.P : v;  // v < ND P
    const bool neg = v > ms.P / 2;                                   // centred [c]_P = neg ? v - P : v
    const W rm = reduce_u64<A>(neg ? ms.P - v : v, c, j);
    const W t = neg ? x[0][i] + rm : x[0][i] + (q - rm);              // (c - [c]_P) mod q, in [0, 2q)
    const W out = A::canon_gs(A::mul4(t, pinv, q), q);
    if (!isb) {
      a_out[(ct * Lk + j) * N + e] = out;
    } else {
      b_out[(size_t)oi * Lk + j] = out;
      if (j == 0 && y0 != nullptr && rs != nullptr) {  // (with em, k_mask_encode wrote y0)
        const uint64_t tm = (1ull << c.t_bits) - 1;
        y0[oi] = (tm + 1 - rs[e]) & tm;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// A3 packing: kernel [M][C][kh][kw] (< 2^t) -> mirrored coefficient-domain polys
// w[m][g][j][O - c*Hw*Ww - l*Ww - l'] = lift_j(K[m, g*Cw+c, l, l']) (reading R3: centred lift).
// The target must be zero-filled before.
template <class W>
__global__ void k_pack_weights(const uint64_t* __restrict__ kern, W* __restrict__ w,
                               const __grid_constant__ DevConsts c, PlanDev pl) {
  const size_t total = (size_t)pl.M * pl.C * pl.kh0 * pl.kw0;
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint32_t l2 = idx % pl.kw0;
  const uint32_t l = (idx / pl.kw0) % pl.kh0;
  const uint32_t ch = (idx / ((size_t)pl.kw0 * pl.kh0)) % pl.C;
  const uint32_t m = idx / ((size_t)pl.kw0 * pl.kh0 * pl.C);
  // polyphase (reading R7b): tap (l, l2) of channel ch is tap (l / s, l2 / s) of phase channel
  // (ch s + l % s) s + l2 % s; ps = 1 leaves everything as it is
  const uint32_t s = pl.ps;
  const uint32_t ce = (ch * s + l % s) * s + l2 % s, a = l / s, b = l2 / s;
  const uint32_t g = ce / pl.Cw, cc = ce % pl.Cw;
  const uint32_t coef = pl.O - cc * pl.Hw * pl.Ww - a * pl.Ww - b;
  const uint64_t t = 1ull << c.t_bits;
  const uint64_t v = kern[idx] & (t - 1);
  const size_t N = 1ull << c.log_n;
  for (uint32_t j = 0; j < c.L; ++j) {
    const uint64_t q = c.q[j];
    const uint64_t lifted = v >= t / 2 ? (q - (t - v) % q) % q : v % q;
    w[(((size_t)m * pl.G + g) * c.L + j) * N + coef] = (W)lifted;
  }
}

// f3 packing: W [n_o][n_i] (< 2^t) -> w[m][g][j][d*nib + nib - 1 - i] = lift_j(W[m*nob + d][g*nib + i])
// (reading R15, the matrix-vector packing; centred lift R3). One thread per matrix entry.
template <class W>
__global__ void k_pack_fc_weights(const uint64_t* __restrict__ Wm, W* __restrict__ w,
                                  const __grid_constant__ DevConsts c, PlanDev pl) {
  const size_t total = (size_t)pl.no * pl.C;
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint32_t col = idx % pl.C, o = idx / pl.C;
  const uint32_t m = o / pl.nob, d = o % pl.nob, g = col / pl.nib, i = col % pl.nib;
  const uint32_t coef = d * pl.nib + pl.nib - 1 - i;
  const uint64_t t = 1ull << c.t_bits;
  const uint64_t v = Wm[idx] & (t - 1);
  const size_t N = 1ull << c.log_n;
  for (uint32_t j = 0; j < c.L; ++j) {
    const uint64_t q = c.q[j];
    const uint64_t lifted = v >= t / 2 ? (q - (t - v) % q) % q : v % q;
    w[(((size_t)m * pl.G + g) * c.L + j) * N + coef] = (W)lifted;
  }
}

// A6 / A7 standalone: ct [n][2][L][N], b_j += enc_j(v[n][N]).
template <class A>
__global__ void k_enc_add(typename A::W* __restrict__ ct, const uint64_t* __restrict__ v,
                          const __grid_constant__ DevConsts c, size_t n) {
  using W = typename A::W;
  const size_t N = 1ull << c.log_n;
  const size_t total = n * c.L * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t e = idx % N;
    const uint32_t j = (idx / N) % c.L;
    const size_t i = idx / (N * c.L);
    W* b = ct + ((i * 2 + 1) * c.L + j) * N + e;
    const uint64_t q = c.q[j];
    const uint64_t s = (uint64_t)*b + (uint64_t)enc_mod<A>(v[i * N + e], EncK(c, j));  // [0, 2q)
    *b = (W)(s >= q ? s - q : s);
  }
}

// Reading R17: the server's mask drawn on the device from Philox4x32-10 (Salmon et al., SC'11),
// counter (e >> 1, ct0 + ct, stream, 0), key (seed lo, seed hi); one draw gives the mask words of
// the coefficient pair (e, e + 1): r[e] = (w1 2^32 + w0) mod 2^t, r[e + 1] = (w3 2^32 + w2) mod 2^t.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int rnd = 0; rnd < 10; ++rnd) {
    if (rnd) k0 += 0x9E3779B9u, k1 += 0xBB67AE85u;
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// r [n_ct][N]: one thread per coefficient pair, 16-byte stores. It reads nothing another kernel
// writes, so it lets its dependents launch at once; it waits for its predecessor only at the end,
// so that its own completion implies the predecessor's (the chain fwd NTT -> draw -> MAC relies on
// this: the MAC's dependency wait then covers the forward NTT's output too).
__global__ void k_mask_draw(uint64_t* __restrict__ r, MaskGen g, size_t n_pairs, uint32_t half_n, uint32_t t_bits) {
  pdl_trigger();
  const uint64_t tm = (1ull << t_bits) - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n_pairs; i += (size_t)gridDim.x * blockDim.x) {
    const uint32_t ct = (uint32_t)(i / half_n), pe = (uint32_t)(i % half_n);
    const uint4 w = philox4x32_10(make_uint4(pe, g.ct0 + ct, g.stream, 0u), (uint32_t)g.seed, (uint32_t)(g.seed >> 32));
    reinterpret_cast<ulonglong2*>(r)[i] =
        make_ulonglong2((((uint64_t)w.y << 32) | w.x) & tm, (((uint64_t)w.w << 32) | w.z) & tm);
  }
  pdl_wait();
}

// A7 prepared once per layer call (the full calls; the stage calls encode r in the tail): the
// encoded mask em[ct][j][e] = enc_j(r[ct][e]) of every output ciphertext the call computes, for
// every limb, with r read from the caller's buffer or drawn from the generator (reading R17); and
// the server's share y0 = -r mod t at the designated outputs (A8). The limb-independent half of
// enc (rho, up) is computed once per coefficient. Launched right after the forward NTT with the
// same chaining as k_mask_draw (it reads nothing the NTT writes; it waits for it at the end), so
// it runs on the SMs the forward NTT leaves idle, and the INTT tails only add em_j (4 or 8 bytes
// per limb-coefficient) instead of reading and encoding r (8 bytes per coefficient, per limb).
// wait_first: a standalone call (secn_mask_encode), whose r may come from the preceding kernel,
// waits for it before reading; chained after the forward NTT it waits only at the end.
// A thread owns MASK_COEFS consecutive coefficients of one output ciphertext (two Philox draws):
// the per-limb constants are loaded once per 4 coefficients and each limb is one 16-byte
// (32-bit words) store. y0 is written by the thread that holds the designated coefficient, from
// the value it already drew (the designation inverted: d = e - O = ii Ww + jj, ii < dh, jj < dw;
// the division by Ww by a multiply-shift that is exact for d < 2^12 <= 2^24 / Ww).
constexpr int MASK_COEFS = 4;

__device__ __forceinline__ uint32_t div_small(uint32_t d, uint32_t magic) { return (uint32_t)(((uint64_t)d * magic) >> 24); }

template <class A>
__global__ void __launch_bounds__(256) k_mask_encode(typename A::W* __restrict__ em, uint64_t* __restrict__ y0,
                                                     const uint64_t* __restrict__ r, MaskGen g,
                                                     const __grid_constant__ DevConsts c,
                                                     const __grid_constant__ PlanDev pl, uint32_t n_act,
                                                     int wait_first) {
  using W = typename A::W;
  pdl_trigger();
  if (wait_first) pdl_wait();
  const uint32_t N = 1u << c.log_n, L = c.L;
  const uint64_t tm = (1ull << c.t_bits) - 1, thalf = 1ull << (c.t_bits - 1);
  // grid (coefficients / (256 MASK_COEFS), active cts): the ct uniform per CTA
  const uint32_t e0 = (blockIdx.x * blockDim.x + threadIdx.x) * MASK_COEFS;
  if (blockIdx.y < n_act && e0 < N) {
    const uint32_t ct = slice_ct(pl, blockIdx.y);
    uint64_t v[MASK_COEFS];
    if (r != nullptr) {
#pragma unroll
      for (int h = 0; h < MASK_COEFS / 2; ++h) {
        const ulonglong2 rr = reinterpret_cast<const ulonglong2*>(r + (size_t)ct * N + e0)[h];
        v[2 * h] = rr.x, v[2 * h + 1] = rr.y;
      }
    } else {
#pragma unroll
      for (int h = 0; h < MASK_COEFS / 2; ++h) {
        const uint4 w = philox4x32_10(make_uint4((e0 >> 1) + h, g.ct0 + ct, g.stream, 0u), (uint32_t)g.seed,
                                      (uint32_t)(g.seed >> 32));
        v[2 * h] = (((uint64_t)w.y << 32) | w.x) & tm, v[2 * h + 1] = (((uint64_t)w.w << 32) | w.z) & tm;
      }
    }
    uint64_t rho[MASK_COEFS];
    uint32_t up[MASK_COEFS];
#pragma unroll
    for (int i = 0; i < MASK_COEFS; ++i) rho[i] = (c.qmt * v[i]) & tm, up[i] = rho[i] >= thalf;
#pragma unroll
    for (uint32_t j = 0; j < SECN_MAX_LIMBS; ++j) {
      if (j >= L) break;
      const EncK ek(c, (int)j);
      W* dst = em + ((size_t)ct * L + j) * N + e0;
      W e[MASK_COEFS];
#pragma unroll
      for (int i = 0; i < MASK_COEFS; ++i) e[i] = enc_limb<A>(rho[i], up[i], ek);
      if constexpr (sizeof(W) == 4) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(e[0], e[1], e[2], e[3]);
      } else {
        reinterpret_cast<ulonglong2*>(dst)[0] = make_ulonglong2(e[0], e[1]);
        reinterpret_cast<ulonglong2*>(dst)[1] = make_ulonglong2(e[2], e[3]);
      }
    }
    if (y0 != nullptr) {  // A8: this thread's designated coefficients (at most MASK_COEFS)
      if (pl.kind == 1) {  // fc: output row m nob + d at coefficient d nib + nib - 1 of output ct m
#pragma unroll
        for (int i = 0; i < MASK_COEFS; ++i) {
          const uint32_t e = e0 + i, d = (e + 1) / pl.nib - 1;
          if ((e + 1) % pl.nib == 0 && d < pl.nob && ct * pl.nob + d < pl.no)
            y0[(size_t)ct * pl.nob + d] = (tm + 1 - v[i]) & tm;
        }
      } else if (e0 + MASK_COEFS > pl.O) {
        const uint32_t dh = pl.Hw - pl.kh + 1, dw = pl.Ww - pl.kw + 1;
        const uint32_t m = ct / pl.S, sidx = ct % pl.S, bh = sidx / pl.nbw, bw = sidx - bh * pl.nbw;
        const uint32_t magic = ((1u << 24) + pl.Ww - 1) / pl.Ww;
#pragma unroll
        for (int i = 0; i < MASK_COEFS; ++i) {
          const uint32_t e = e0 + i;
          if (e < pl.O) continue;
          const uint32_t d = e - pl.O, ii = div_small(d, magic), jj = d - ii * pl.Ww;
          if (ii >= dh || jj >= dw) continue;
          const uint32_t py = bh * dh + ii, px = bw * dw + jj, oy = py / pl.sh, ox = px / pl.sh;
          if (oy * pl.sh != py || ox * pl.sh != px || oy >= pl.OH || ox >= pl.OW) continue;
          y0[((size_t)m * pl.OH + oy) * pl.OW + ox] = (tm + 1 - v[i]) & tm;
        }
      }
    }
  }
  if (!wait_first) pdl_wait();
}

// Designated server share y0[m][oy][ox] = (t - r[m*S+s][O + i*Ww + j]) mod t.
__global__ void k_extract_share(const uint64_t* __restrict__ r, uint64_t* __restrict__ y0,
                                const __grid_constant__ DevConsts c, PlanDev pl) {
  pdl_wait();
  pdl_trigger();
  const size_t total = (size_t)pl.M * pl.OH * pl.OW;
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint32_t ox = idx % pl.OW, oy = (idx / pl.OW) % pl.OH, m = idx / ((size_t)pl.OW * pl.OH);
  const uint32_t py = oy * pl.sh, px = ox * pl.sh;
  const uint32_t bh = py / (pl.Hw - pl.kh + 1), i = py % (pl.Hw - pl.kh + 1);
  const uint32_t bw = px / (pl.Ww - pl.kw + 1), jj = px % (pl.Ww - pl.kw + 1);
  const uint32_t s = bh * pl.nbw + bw;
  if (s < pl.s0 || s >= pl.s0 + pl.sn) return;  // another call's spatial slice
  const size_t N = 1ull << c.log_n;
  const uint64_t t = 1ull << c.t_bits;
  y0[idx] = (t - r[((size_t)m * pl.S + s) * N + pl.O + i * pl.Ww + jj]) & (t - 1);
}

// SECN_VALIDATE: kind 0 = residues (limb = (idx / N) mod L, must be < q_j), kind 1 = uint64
// plaintext-side values (must be < 2^t_bits). Sets *flag on a violation.
template <class W>
__global__ void k_check_range(const W* __restrict__ v, size_t n_words, const __grid_constant__ DevConsts c,
                              int kind, uint32_t* flag) {
  const size_t N = 1ull << c.log_n;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n_words; idx += (size_t)gridDim.x * blockDim.x) {
    const uint64_t bound = kind == 0 ? c.q[(idx / N) % c.L] : (1ull << c.t_bits);
    if ((uint64_t)v[idx] >= bound) *flag = 1;
  }
}

// ------------------------------------------------------------------------------------------
// launchers

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

void read_tune(int device, Tune* t) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms <= 0) sms = 148;
  t->num_sms = sms;
  t->no_pdl = env_int("SECN_NO_PDL", 0);
  t->ntt_np2_min = env_int("SECN_NTT_NP2_MIN", 2 * sms * 6);
  t->ntt_tma = env_int("SECN_NTT_TMA", 1);
  t->ntt_tma_min = env_int("SECN_NTT_TMA_MIN", 0);
  t->tail1 = env_int("SECN_TAIL1", 0);
  t->mac_kb = env_int("SECN_MAC_KB", 110);
  t->mac_xamort = env_int("SECN_MAC_XAMORT", 1);
  t->mac_nmr = env_int("SECN_MAC_NMR", 0);
  t->mac_nohint = env_int("SECN_MAC_NOHINT", 0);
  t->mac_pre = env_int("SECN_MAC_PRE", 2);
  t->mac_sg = env_int("SECN_MAC_SG", 0);
  t->mac_mt = env_int("SECN_MAC_MT", 0);
  t->fused = env_int("SECN_FUSED", 0);
  t->mac_ws = env_int("SECN_MAC_WS", 1);
  t->fused_sg = env_int("SECN_FUSED_SG", 0);
  t->fused_mt = env_int("SECN_FUSED_MT", 0);
  t->fused_kb = env_int("SECN_FUSED_KB", 112);
  t->validate = env_int("SECN_VALIDATE", 0);
}

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while the
// preceding kernel in the stream finishes; it synchronises with pdl_wait() before reading that
// kernel's outputs. Captured into CUDA graphs as programmatic edges.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(const DevConsts& c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c.tune.no_pdl ? 0 : 1;  // SECN_NO_PDL=1: plain stream order (debugging)
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Launch geometry of the NTT kernels: NP = 2 (two polys of one limb per CTA, shared twiddles)
// for 32-bit limbs at N = 4096 when the batch has an even poly count and fills the GPU several
// times over; otherwise NP = 1. Both poly-index parities (ct, component) are preserved.
template <class A, int LOGN, int NP>
static cudaError_t ntt_fwd_np(const DevConsts& c, const void* in, void* out, size_t n_polys, const uint64_t* x0,
                              cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  const size_t smem = (size_t)NP * smem_words<LOGN>() * sizeof(W);  // opted in by init_device
  // groups per launch: an even number so that x0's ct index stays (poly index) / 2
  const size_t gmax = (0x7fffffffull / c.L) & ~(size_t)1;
  const size_t ngroups = n_polys / NP;
  for (size_t g0 = 0; g0 < ngroups; g0 += gmax) {
    const size_t ng = ngroups - g0 < gmax ? ngroups - g0 : gmax;
    const size_t off = g0 * NP * c.L * N;
    const W* src = static_cast<const W*>(in) + off;
    W* dst = static_cast<W*>(out) + off;
    const uint64_t* xs = x0 ? x0 + g0 * NP / 2 * N : nullptr;
    cudaError_t e = launch_pdl(c, k_ntt_fwd<A, LOGN, NP>, dim3((unsigned)(ng * c.L)), dim3(N / 16), smem, s, src, dst, c, xs);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <class A, int LOGN, int NP>
static cudaError_t ntt_inv_np(const DevConsts& c, void* polys, size_t n_polys, cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  const size_t smem = (size_t)NP * smem_words<LOGN>() * sizeof(W);  // opted in by init_device
  const size_t gmax = (0x7fffffffull / c.L) & ~(size_t)1;
  const size_t ngroups = n_polys / NP;
  for (size_t g0 = 0; g0 < ngroups; g0 += gmax) {
    const size_t ng = ngroups - g0 < gmax ? ngroups - g0 : gmax;
    W* buf = static_cast<W*>(polys) + g0 * NP * c.L * N;
    cudaError_t e = launch_pdl(c, k_ntt_inv<A, LOGN, NP>, dim3((unsigned)(ng * c.L)), dim3(N / 16), smem, s, buf, c);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

static bool encode_tmap(CUtensorMap* m, int wb, int rank, const void* base, const cuuint64_t* dims,
                        const cuuint64_t* strides_bytes, const cuuint32_t* box, bool swizzle128 = false);

// the TMA-staged engine (k_ntt_tma): polys [n_polys][L][N] viewed as (128-byte row, row, limb,
// poly); persistent grid of L x per_limb CTAs (ntt_tma_minb per SM)
template <class A, int LOGN, bool INV>
static cudaError_t ntt_tma(const DevConsts& c, const void* in, void* out, size_t n_polys, cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN, NP = ntt_tma_np<A, LOGN>();
  constexpr int RW = 128 / (int)sizeof(W), ROWS = N / RW, BR = ROWS < 256 ? ROWS : 256;
  const size_t pmax = (size_t)1 << 30;  // polys per launch (32-bit TMA coordinates)
  for (size_t p0 = 0; p0 < n_polys; p0 += pmax) {
    const size_t np = n_polys - p0 < pmax ? n_polys - p0 : pmax;
    const size_t off = p0 * c.L * N;
    CUtensorMap tm;
    const cuuint64_t d[4] = {(cuuint64_t)RW, (cuuint64_t)ROWS, c.L, np};
    const cuuint64_t st[3] = {128, (cuuint64_t)N * sizeof(W), (cuuint64_t)c.L * N * sizeof(W)};
    const cuuint32_t box[4] = {(cuuint32_t)RW, (cuuint32_t)BR, 1, 1};
    CUtensorMap tmo;  // the output (in place: the same tensor)
    if (!encode_tmap(&tm, (int)sizeof(W), 4, static_cast<const W*>(in) + off, d, st, box, true) ||
        !encode_tmap(&tmo, (int)sizeof(W), 4, static_cast<W*>(out) + off, d, st, box, true))
      return cudaErrorInvalidValue;
    const size_t items = (np + NP - 1) / NP;
    size_t per_limb = (size_t)ntt_tma_minb<A, LOGN>() * c.tune.num_sms / c.L;
    per_limb = per_limb < 1 ? 1 : per_limb > items ? items : per_limb;
    cudaError_t e = launch_pdl(c, k_ntt_tma<A, LOGN, INV>, dim3((unsigned)(per_limb * c.L)), dim3(N / 16),
                               ntt_tma_smem<A, LOGN>(), s, tm, tmo, static_cast<W*>(out) + off, c, (uint32_t)np);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Which plain calls take the TMA-staged engine (SECN_NTT_TMA: 0 never, 1 this rule, 2 always):
// the shapes where it measured faster on the C5 sweep (profiles/r02t_*, r02z_*): the 32-bit
// N = 4096 forward (with its TMA store: 0.50 of HBM against 0.485), every inverse except 32-bit
// N = 4096 with an even poly count (the two-poly one-CTA-per-poly kernel at 4 CTAs per SM is 2%
// faster there), the 32-bit N = 4096 inverse with an odd count (where the old kernels fall back
// to one poly per CTA: 0.38 -> 0.49), and both directions at 32-bit N = 2^14 and 64-bit 2^13.
template <class A, int LOGN, bool INV>
static bool use_ntt_tma(const DevConsts& c, size_t n_polys, size_t P) {
  if (c.tune.ntt_tma == 0 || P < (size_t)c.tune.ntt_tma_min) return false;
  if (c.tune.ntt_tma == 2) return true;
  constexpr bool w32 = sizeof(typename A::W) == 4;
  if (w32 && LOGN == 12) return !INV || n_polys % 2 == 1;
  if (w32 && LOGN == 14) return true;
  if (!w32 && LOGN == 13) return true;
  return INV;
}

template <class A, int LOGN>
static cudaError_t ntt_fwd_t(const DevConsts& c, const void* in, void* out, size_t P, const uint64_t* x0,
                             cudaStream_t s) {
  const size_t n_polys = P / c.L;
  if (x0 == nullptr && use_ntt_tma<A, LOGN, false>(c, n_polys, P)) return ntt_tma<A, LOGN, false>(c, in, out, n_polys, s);
  if constexpr (sizeof(typename A::W) == 4 && LOGN == 12)
    if (n_polys % 2 == 0 && P >= (size_t)c.tune.ntt_np2_min) return ntt_fwd_np<A, LOGN, 2>(c, in, out, n_polys, x0, s);
  return ntt_fwd_np<A, LOGN, 1>(c, in, out, n_polys, x0, s);
}

template <class A, int LOGN>
static cudaError_t ntt_inv_t(const DevConsts& c, void* polys, size_t P, cudaStream_t s) {
  const size_t n_polys = P / c.L;
  if (use_ntt_tma<A, LOGN, true>(c, n_polys, P)) return ntt_tma<A, LOGN, true>(c, polys, polys, n_polys, s);
  if constexpr (sizeof(typename A::W) == 4 && LOGN == 12)
    if (n_polys % 2 == 0 && P >= (size_t)c.tune.ntt_np2_min) return ntt_inv_np<A, LOGN, 2>(c, polys, n_polys, s);
  return ntt_inv_np<A, LOGN, 1>(c, polys, n_polys, s);
}

template <class A, int LOGN>
static cudaError_t ntt_inv_tail_t(const DevConsts& c, void* polys, size_t P, const uint64_t* r, uint64_t* y0,
                                  const PlanDev& pl, cudaStream_t s, bool chained, const void* emv) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  const size_t smem = LOGN > 12 ? smem_words<LOGN>() * sizeof(W) : 0;  // opted in by init_device
  const int r_early = chained ? 1 : 0;
  const size_t pmax = (0x7fffffffull / c.L / 2) * 2;  // polys per launch: even, so r's index is p/2
  const size_t n_polys = P / c.L;
  for (size_t p0 = 0; p0 < n_polys; p0 += pmax) {
    const size_t np = n_polys - p0 < pmax ? n_polys - p0 : pmax;
    // with an s-slice the chunk's rows start at row p0 / 2 (rows >= active index, see slice_ct)
    W* buf = static_cast<W*>(polys) + p0 * c.L * N;
    const uint64_t* rs = r ? r + p0 / 2 * N : nullptr;
    const W* em = static_cast<const W*>(emv);  // indexed by the global row in the kernels
    cudaError_t e;
    if constexpr (LOGN == 12 && sizeof(W) == 4) {
      if (c.tune.tail1)
        e = launch_pdl(c, k_ntt_inv_tail<A, LOGN>, dim3((unsigned)(np * c.L)), dim3(N / 16), smem, s, buf, c, rs, y0,
                       pl, p0 / 2, r_early, em);
      else if (em != nullptr)  // both components of a (ciphertext, limb) per CTA, by bulk copies
        e = launch_pdl(c, k_ntt_inv_tail_bulk<A>, dim3((unsigned)(np / 2 * c.L)), dim3(256),
                       3 * N * sizeof(W) + 16, s, buf, c, pl, p0 / 2, em);
      else if (r_early)
        e = launch_pdl(c, k_ntt_inv_tail2<A, 1>, dim3((unsigned)(np / 2 * c.L)), dim3(256), 0, s, buf, c, rs, y0, pl,
                       p0 / 2, em);
      else
        e = launch_pdl(c, k_ntt_inv_tail2<A, 0>, dim3((unsigned)(np / 2 * c.L)), dim3(256), 0, s, buf, c, rs, y0, pl,
                       p0 / 2, em);
    } else {
      e = launch_pdl(c, k_ntt_inv_tail<A, LOGN>, dim3((unsigned)(np * c.L)), dim3(N / 16), smem, s, buf, c, rs, y0, pl,
                     p0 / 2, r_early || em != nullptr ? 1 : 0, em);
    }
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_ntt_inv_tail(const DevConsts& c, void* polys, size_t P, const uint64_t* r, uint64_t* y0,
                                const PlanDev& pl, cudaStream_t s, bool chained, const void* em) {
  if (P == 0) return cudaSuccess;
  if (c.word_bits == 64) {
    switch (c.log_n) {
      case 12: return ntt_inv_tail_t<Arith64, 12>(c, polys, P, r, y0, pl, s, chained, em);
      case 13: return ntt_inv_tail_t<Arith64, 13>(c, polys, P, r, y0, pl, s, chained, em);
      case 14: return ntt_inv_tail_t<Arith64, 14>(c, polys, P, r, y0, pl, s, chained, em);
    }
  } else {
    switch (c.log_n) {
      case 12: return ntt_inv_tail_t<Arith32, 12>(c, polys, P, r, y0, pl, s, chained, em);
      case 13: return ntt_inv_tail_t<Arith32, 13>(c, polys, P, r, y0, pl, s, chained, em);
      case 14: return ntt_inv_tail_t<Arith32, 14>(c, polys, P, r, y0, pl, s, chained, em);
    }
  }
  return cudaErrorInvalidValue;
}

// Cluster NTT: one cluster of two CTAs per limb-poly (launches of <= 2^30 polys)
template <class A, int LOGH>
static cudaError_t ntt_cl(const DevConsts& c, const void* in, void* out, size_t P, const uint64_t* x0, bool inverse,
                          cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 2 << LOGH, T = (1 << LOGH) / 16;
  const size_t smem = smem_words<LOGH>() * sizeof(W);  // opted in by init_device
  // polys per launch: a multiple of 2L so that the ct index of x0 stays (poly / L) / 2
  const size_t pmax = ((size_t)1 << 30) / (2 * c.L) * (2 * c.L);
  for (size_t p0 = 0; p0 < P; p0 += pmax) {
    const size_t np = P - p0 < pmax ? P - p0 : pmax;
    const size_t off = p0 * N;
    cudaError_t e;
    if (inverse)
      e = launch_pdl(c, k_ntt_inv_cl<A, LOGH>, dim3((unsigned)(2 * np)), dim3(T), smem, s, static_cast<W*>(out) + off, c);
    else
      e = launch_pdl(c, k_ntt_fwd_cl<A, LOGH>, dim3((unsigned)(2 * np)), dim3(T), smem, s,
                     static_cast<const W*>(in) + off, static_cast<W*>(out) + off, c,
                     x0 ? x0 + p0 / c.L / 2 * N : nullptr);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_ntt_fwd(const DevConsts& c, const void* in, void* out, size_t P, const uint64_t* x0,
                           cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  if (c.log_n == 15)
    return c.word_bits == 64 ? ntt_cl<Arith64, 14>(c, in, out, P, x0, false, s)
                             : ntt_cl<Arith32, 14>(c, in, out, P, x0, false, s);
  if (c.log_n == 14 && c.word_bits == 64) return ntt_cl<Arith64, 13>(c, in, out, P, x0, false, s);
  if (c.word_bits == 64) {
    switch (c.log_n) {
      case 12: return ntt_fwd_t<Arith64, 12>(c, in, out, P, x0, s);
      case 13: return ntt_fwd_t<Arith64, 13>(c, in, out, P, x0, s);
    }
  } else {
    switch (c.log_n) {
      case 12: return ntt_fwd_t<Arith32, 12>(c, in, out, P, x0, s);
      case 13: return ntt_fwd_t<Arith32, 13>(c, in, out, P, x0, s);
      case 14: return ntt_fwd_t<Arith32, 14>(c, in, out, P, x0, s);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_ntt_inv(const DevConsts& c, void* polys, size_t P, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  if (c.log_n == 15)
    return c.word_bits == 64 ? ntt_cl<Arith64, 14>(c, nullptr, polys, P, nullptr, true, s)
                             : ntt_cl<Arith32, 14>(c, nullptr, polys, P, nullptr, true, s);
  if (c.log_n == 14 && c.word_bits == 64) return ntt_cl<Arith64, 13>(c, nullptr, polys, P, nullptr, true, s);
  if (c.word_bits == 64) {
    switch (c.log_n) {
      case 12: return ntt_inv_t<Arith64, 12>(c, polys, P, s);
      case 13: return ntt_inv_t<Arith64, 13>(c, polys, P, s);
    }
  } else {
    switch (c.log_n) {
      case 12: return ntt_inv_t<Arith32, 12>(c, polys, P, s);
      case 13: return ntt_inv_t<Arith32, 13>(c, polys, P, s);
      case 14: return ntt_inv_t<Arith32, 14>(c, polys, P, s);
    }
  }
  return cudaErrorInvalidValue;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link dependency)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static bool encode_tmap(CUtensorMap* m, int wb, int rank, const void* base, const cuuint64_t* dims,
                        const cuuint64_t* strides_bytes, const cuuint32_t* box, bool swizzle128) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, wb == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, rank,
             const_cast<void*>(base), dims, strides_bytes, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// WS: the warp-specialised k_mac_ws (32-bit limbs, two output-chunk buffers) instead of k_mac
template <class W, int SG, int MT, bool WS = false>
static cudaError_t mac_t(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                         cudaStream_t s, bool chained) {
  const int N = 1 << c.log_n;
  const size_t xtile = (size_t)p.G * 2 * SG * MAC_THREADS * sizeof(W);
  const size_t stage = (size_t)MT * MAC_THREADS * sizeof(W);
  // ring depth: fill ~110 KiB per CTA (two CTAs per SM) after the X^ tile, 4..32 stages
  const size_t chunks = (size_t)MT * 2 * SG * MAC_CHS * sizeof(W) * (WS ? 2 : 1) + MAC_THREADS * 2 * sizeof(W);
  const size_t fixed = xtile + chunks + (WS ? 4 * sizeof(uint64_t) : 0);
  const size_t cta_budget = (size_t)c.tune.mac_kb * 1024;
  const size_t budget = cta_budget > fixed + 4 * stage ? cta_budget - fixed : 4 * stage;
  int NS = (int)(budget / stage);
  NS = NS < 4 ? 4 : NS > 32 ? 32 : NS;
  const size_t smem = fixed + NS * stage + (2 * NS + 1) * sizeof(uint64_t);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;  // opted in by init_device
  const int n_sg = (p.sn + SG - 1) / SG;
  // m-range per CTA: the split of M into n_mr ranges (each >= MT channels, a multiple of MT)
  // whose CTA count fills whole waves of two CTAs per SM best; ties go to fewer, longer CTAs
  // (each CTA pays one X^ tile load and one pipeline fill).
  const long ctas_no_m = (long)(N / MAC_THREADS) * n_sg * c.L;
  const long wave = (long)c.tune.num_sms * 2;
  const int mblocks = (p.M + MT - 1) / MT;
  int best_nmr = 1;
  double best_eff = -1.0;
  for (int nmr = 1; nmr <= mblocks; ++nmr) {
    const int per = (mblocks + nmr - 1) / nmr;  // m-blocks per CTA
    const int used = (mblocks + per - 1) / per;
    if (used != nmr) continue;
    const long ctas = (long)nmr * ctas_no_m;
    const long waves = (ctas + wave - 1) / wave;
    const double eff = (double)ctas / (double)(waves * wave) - 0.02 * (double)waves;
    if (eff > best_eff + 1e-9) best_eff = eff, best_nmr = nmr;
  }
  // layers with few input groups or few output channels: one m-block per CTA (more, shorter CTAs
  // hide the INTT-level latency better; measured on the SqueezeNet fire layers)
  if (WS)  // the pipeline needs >= 2 m-blocks per CTA (its MAC of one overlaps the INTT of the last)
    best_nmr = best_nmr < (mblocks + 1) / 2 ? best_nmr : (mblocks + 1) / 2;
  else if ((p.G <= 4 && p.M < 256) || p.M <= 48)  // (G <= 4 with M >= 256: the wave-fill split,
    best_nmr = mblocks;                               //  several m-blocks per CTA; profiles/r02zq_*)
  else if (xtile >= (size_t)MT * p.G * MAC_THREADS * sizeof(W) && c.tune.mac_xamort)
    // the X^ tile is at least one m-block of weights: a CTA takes >= 2 m-blocks so the tile load
    // is amortised (conv1 of SqueezeNet-1.1: 79 -> 69 us)
    best_nmr = best_nmr < (mblocks + 1) / 2 ? best_nmr : (mblocks + 1) / 2;
  if (const int nmr_env = c.tune.mac_nmr) best_nmr = nmr_env < mblocks ? nmr_env : mblocks;
  const int m_range = ((mblocks + best_nmr - 1) / best_nmr) * MT;
  const int n_mr = (p.M + m_range - 1) / m_range;
  // tensor maps: X^ [G][S*2][L][N] viewed as (N, L, 2S, G); W [M][G][L][N] as (N, G*L, M)
  const cuuint64_t wb = sizeof(W);
  CUtensorMap tmx, tmw;
  const cuuint64_t xd[4] = {(cuuint64_t)N, c.L, 2ull * p.S, p.G};
  const cuuint64_t xs_[3] = {N * wb, (cuuint64_t)c.L * N * wb, 2ull * p.S * c.L * N * wb};
  const cuuint32_t xb[4] = {MAC_THREADS, 1, 2 * SG, p.G};
  const cuuint64_t wd[3] = {(cuuint64_t)N, (cuuint64_t)p.G * c.L, p.M};
  const cuuint64_t ws_[2] = {N * wb, (cuuint64_t)p.G * c.L * N * wb};
  const cuuint32_t wbx[3] = {MAC_THREADS, 1, MT};
  if (!encode_tmap(&tmx, (int)wb, 4, xhat, xd, xs_, xb) || !encode_tmap(&tmw, (int)wb, 3, w, wd, ws_, wbx))
    return cudaErrorInvalidValue;
  dim3 grid((N / MAC_THREADS) * n_sg, c.L, n_mr);
  W* yp = static_cast<W*>(y);
  DevConsts cc = c;  // debugging knobs ride in unused word_bits bits
  if (c.tune.mac_nohint) cc.word_bits |= 0x400;
  // ring stages issued before the dependency wait (and the X^ tile): only when the preceding
  // launch is this call's forward NTT, which never writes the weights (internal.h, "Pre-wait reads")
  const int n_pre = chained ? c.tune.mac_pre : 0;
  cudaError_t e;
  if constexpr (WS)
    e = launch_pdl(c, k_mac_ws<SG, MT>, grid, dim3(MAC_THREADS + 32), smem, s, tmx, tmw, yp, cc, p, m_range, n_sg, NS,
                   n_pre);
  else
    e = launch_pdl(c, k_mac<W, SG, MT>, grid, dim3(MAC_THREADS + 32), smem, s, tmx, tmw, yp, cc, p, m_range, n_sg, NS,
                   n_pre);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_mac(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                       cudaStream_t s, bool chained) {
  if (p.M == 0 || p.S == 0) return cudaSuccess;
  if (p.G > 32) return cudaErrorInvalidValue;
  // s-group: among the SG <= 4 whose X^ tile fits in 64 KiB, the one minimising
  // n_sg (SG + 1/2), n_sg = ceil(S / SG): the MAC work including zero-padded blocks plus half a
  // block per pass over the weights (fitted to the per-layer sweep in profiles/); ties go to the
  // smaller SG. Accumulator block MT x 2SG <= 32 64-bit sums (32-bit limbs) or <= 12 128-bit sums
  // (64-bit limbs), spill-free at the 96 registers two 288-thread CTAs per SM allow.
  const size_t wb = c.word_bits / 8;
  int sg = 1;
  for (int cand = 2; cand <= 4 && cand <= (int)p.sn; ++cand) {
    if ((size_t)p.G * 2 * cand * MAC_THREADS * wb > 64 * 1024) break;
    const int nc = (int)((p.sn + cand - 1) / cand), nb = (int)((p.sn + sg - 1) / sg);
    if (nc * (2 * cand + 1) < nb * (2 * sg + 1)) sg = cand;
  }
  if (const int sg_env = c.tune.mac_sg) sg = sg_env;
  if (c.word_bits == 32) {
    // output channels per m-block: the larger register block (more weight reuse) unless its
    // staged chunks plus a 4-stage ring would leave one CTA per SM; then the smaller one
    // (SG = 1 also takes the smaller block once the X^ tile exceeds 24 KiB: measured on conv10)
    static const int mt_big[5] = {0, 16, 8, 5, 3}, mt_small[5] = {0, 8, 4, 2, 2};
    const size_t xtile = (size_t)p.G * 2 * sg * MAC_THREADS * wb;
    const auto fits2 = [&](int mt) {
      const size_t chunks = (size_t)mt * 2 * sg * MAC_CHS * wb + MAC_THREADS * 2 * wb;
      return xtile + chunks + 4 * (size_t)mt * MAC_THREADS * wb <= 110 * 1024;
    };
    bool small = !fits2(mt_big[sg]) || (sg == 1 && xtile > 24 * 1024);
    if (const int mt_env = c.tune.mac_mt) small = mt_env == mt_small[sg];
    // the warp-specialised pipeline (k_mac_ws) where its two phases balance: measured per layer on
    // SqueezeNet-1.1 and ResNet-50 (profiles/r02_mac_ws_ab_*.txt): faster for one s-group, 5..22
    // input groups and >= 48 channels (a tiny MAC phase, G <= 4 with M >= 256, leaves half its warps
    // idle; a long one, G >= 25 or several s-groups, needs all eight); SECN_MAC_WS=0/2: never/always
    const bool ws_rule = sg == 1 && p.G <= 22 && p.M >= 48 && !(p.G <= 4 && p.M >= 256);
    if ((c.tune.mac_ws == 2 || (c.tune.mac_ws == 1 && ws_rule)) && (size_t)p.M > (size_t)mt_small[sg]) {
      switch (sg) {
        case 1: return mac_t<uint32_t, 1, 8, true>(c, p, xhat, w, y, s, chained);
        case 2: return mac_t<uint32_t, 2, 4, true>(c, p, xhat, w, y, s, chained);
        case 3: return mac_t<uint32_t, 3, 2, true>(c, p, xhat, w, y, s, chained);
        default: return mac_t<uint32_t, 4, 2, true>(c, p, xhat, w, y, s, chained);
      }
    }
    if (small) {
      switch (sg) {
        case 1: return mac_t<uint32_t, 1, 8>(c, p, xhat, w, y, s, chained);
        case 2: return mac_t<uint32_t, 2, 4>(c, p, xhat, w, y, s, chained);
        case 3: return mac_t<uint32_t, 3, 2>(c, p, xhat, w, y, s, chained);
        default: return mac_t<uint32_t, 4, 2>(c, p, xhat, w, y, s, chained);
      }
    }
    switch (sg) {
      case 1: return mac_t<uint32_t, 1, 16>(c, p, xhat, w, y, s, chained);
      case 2: return mac_t<uint32_t, 2, 8>(c, p, xhat, w, y, s, chained);
      case 3: return mac_t<uint32_t, 3, 5>(c, p, xhat, w, y, s, chained);
      default: return mac_t<uint32_t, 4, 3>(c, p, xhat, w, y, s, chained);
    }
  }
  switch (sg) {
    case 1: return mac_t<uint64_t, 1, 4>(c, p, xhat, w, y, s, chained);
    case 2: return mac_t<uint64_t, 2, 2>(c, p, xhat, w, y, s, chained);
    case 3: return mac_t<uint64_t, 3, 2>(c, p, xhat, w, y, s, chained);
    default: return mac_t<uint64_t, 4, 1>(c, p, xhat, w, y, s, chained);
  }
}

// Per-device opt-in of the dynamic shared memory every launcher may request (function attributes
// belong to the device that is current when they are set; secn_ctx_create runs this on its
// device, so launches never set attributes and need no process-global state).
template <class K>
static cudaError_t optin(K* kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

cudaError_t init_device(uint32_t word_bits) {
  int dev = 0, optin_max = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const int b = optin_max;
  cudaError_t r = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (r == cudaSuccess) r = x;
  };
  if (word_bits == 64) {
    using A = Arith64;
    chk(optin(k_ntt_fwd<A, 12, 1>, b)), chk(optin(k_ntt_fwd<A, 13, 1>, b));
    chk(optin(k_ntt_inv<A, 12, 1>, b)), chk(optin(k_ntt_inv<A, 13, 1>, b));
    chk(optin(k_ntt_inv_tail<A, 12>, b)), chk(optin(k_ntt_inv_tail<A, 13>, b)), chk(optin(k_ntt_inv_tail<A, 14>, b));
    chk(optin(k_ntt_tma<A, 12, false>, b)), chk(optin(k_ntt_tma<A, 12, true>, b));
    chk(optin(k_ntt_tma<A, 13, false>, b)), chk(optin(k_ntt_tma<A, 13, true>, b));
    chk(optin(k_ntt_fwd_cl<A, 13>, b)), chk(optin(k_ntt_inv_cl<A, 13>, b));
    chk(optin(k_ntt_fwd_cl<A, 14>, b)), chk(optin(k_ntt_inv_cl<A, 14>, b));
    chk(optin(k_mac<uint64_t, 1, 4>, b)), chk(optin(k_mac<uint64_t, 2, 2>, b));
    chk(optin(k_mac<uint64_t, 3, 2>, b)), chk(optin(k_mac<uint64_t, 4, 1>, b));
  } else {
    using A = Arith32;
    chk(optin(k_ntt_fwd<A, 12, 1>, b)), chk(optin(k_ntt_fwd<A, 12, 2>, b));
    chk(optin(k_ntt_fwd<A, 13, 1>, b)), chk(optin(k_ntt_fwd<A, 14, 1>, b));
    chk(optin(k_ntt_inv<A, 12, 1>, b)), chk(optin(k_ntt_inv<A, 12, 2>, b));
    chk(optin(k_ntt_inv<A, 13, 1>, b)), chk(optin(k_ntt_inv<A, 14, 1>, b));
    chk(optin(k_ntt_inv_tail<A, 12>, b)), chk(optin(k_ntt_inv_tail<A, 13>, b)), chk(optin(k_ntt_inv_tail<A, 14>, b));
    chk(optin(k_ntt_tma<A, 12, false>, b)), chk(optin(k_ntt_tma<A, 12, true>, b));
    chk(optin(k_ntt_tma<A, 13, false>, b)), chk(optin(k_ntt_tma<A, 13, true>, b));
    chk(optin(k_ntt_tma<A, 14, false>, b)), chk(optin(k_ntt_tma<A, 14, true>, b));
    chk(optin(k_ntt_inv_tail_bulk<A>, b));
    chk(optin(k_ntt_fwd_cl<A, 14>, b)), chk(optin(k_ntt_inv_cl<A, 14>, b));
    chk(optin(k_mac<uint32_t, 1, 16>, b)), chk(optin(k_mac<uint32_t, 2, 8>, b));
    chk(optin(k_mac<uint32_t, 3, 5>, b)), chk(optin(k_mac<uint32_t, 4, 3>, b));
    chk(optin(k_mac<uint32_t, 1, 8>, b)), chk(optin(k_mac<uint32_t, 2, 4>, b));
    chk(optin(k_mac<uint32_t, 3, 2>, b)), chk(optin(k_mac<uint32_t, 4, 2>, b));
    chk(optin(k_mac_ws<1, 8>, b)), chk(optin(k_mac_ws<2, 4>, b)), chk(optin(k_mac_ws<3, 2>, b));
    chk(optin(k_mac_ws<4, 2>, b));
    chk(optin(k_layer_fused<1, 1>, b)), chk(optin(k_layer_fused<1, 2>, b)), chk(optin(k_layer_fused<1, 4>, b));
    chk(optin(k_layer_fused<2, 1>, b)), chk(optin(k_layer_fused<2, 2>, b));
  }
  return r;
}

// ---- the fused small-layer kernel (k_layer_fused) ----
template <int SG, int MT>
static size_t fused_smem(const DevConsts& c, int G, int* NS_out, int* GC_out) {
  constexpr int A2 = 2 * SG, NP = MT * A2;
  const size_t obuf = (size_t)NP * smem_words<12>() * sizeof(uint32_t);
  const size_t per_g = (size_t)(A2 + MT) * FUSED_THREADS * sizeof(uint32_t);
  const size_t budget = (size_t)c.tune.fused_kb * 1024;
  const size_t ring = budget > obuf + 2 * per_g ? budget - obuf : 2 * per_g;
  int GC = (int)(ring / (2 * per_g));
  GC = GC < 1 ? 1 : GC > G ? G : GC;
  int NS = (int)(ring / (GC * per_g));
  NS = NS < 2 ? 2 : NS > 4 ? 4 : NS;
  *NS_out = NS, *GC_out = GC;
  return obuf + (size_t)NS * GC * per_g + 2 * NS * sizeof(uint64_t);
}

template <int SG, int MT>
static cudaError_t fused_t(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                           const uint64_t* r, uint64_t* y0, cudaStream_t s, bool chained, const void* em) {
  constexpr int N = 4096;
  int NS = 0, GC = 0;
  const size_t smem = fused_smem<SG, MT>(c, (int)p.G, &NS, &GC);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;  // opted in by init_device
  const int n_sg = (p.sn + SG - 1) / SG, n_mb = (p.M + MT - 1) / MT;
  // X^ [G][S*2][L][N] as (N, L, 2S, G); W [M][G][L][N] as (N, L, G, M)
  const cuuint64_t wb = 4;
  CUtensorMap tmx, tmw;
  const cuuint64_t xd[4] = {(cuuint64_t)N, c.L, 2ull * p.S, p.G};
  const cuuint64_t xs_[3] = {N * wb, (cuuint64_t)c.L * N * wb, 2ull * p.S * c.L * N * wb};
  const cuuint32_t xb[4] = {FUSED_THREADS, 1, 2 * SG, (cuuint32_t)GC};
  const cuuint64_t wd[4] = {(cuuint64_t)N, c.L, p.G, p.M};
  const cuuint64_t ws_[3] = {N * wb, (cuuint64_t)c.L * N * wb, (cuuint64_t)p.G * c.L * N * wb};
  const cuuint32_t wbx[4] = {FUSED_THREADS, 1, (cuuint32_t)GC, MT};
  if (!encode_tmap(&tmx, 4, 4, xhat, xd, xs_, xb) || !encode_tmap(&tmw, 4, 4, w, wd, ws_, wbx))
    return cudaErrorInvalidValue;
  const int n_pre = chained ? c.tune.mac_pre : 0;
  cudaError_t e = launch_pdl(c, k_layer_fused<SG, MT>, dim3((unsigned)(n_mb * n_sg), c.L), dim3(FUSED_THREADS + 32),
                             smem, s, tmx, tmw, static_cast<uint32_t*>(y), r, y0, c, p, n_sg, NS, GC, n_pre,
                             static_cast<const uint32_t*>(em));
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool fused_applies(const DevConsts& c, const PlanDev& p) {
  if (c.word_bits != 32 || c.log_n != 12 || p.G > 32 || p.M == 0 || p.S == 0 || c.tune.fused == 0) return false;
  // SECN_FUSED=2: every layer it supports. Off by default: on every SqueezeNet-1.1 layer it measured
  // slower than the three-kernel chain (profiles/r02_fused_ab.txt)
  return c.tune.fused == 2;
}

cudaError_t launch_layer_fused(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                               const uint64_t* r, uint64_t* y0, cudaStream_t s, bool chained, const void* em) {
  int sg = c.tune.fused_sg > 0 ? c.tune.fused_sg : 1;
  int mt = c.tune.fused_mt > 0 ? c.tune.fused_mt : 2;
  if (sg == 1 && mt == 1) return fused_t<1, 1>(c, p, xhat, w, y, r, y0, s, chained, em);
  if (sg == 1 && mt == 2) return fused_t<1, 2>(c, p, xhat, w, y, r, y0, s, chained, em);
  if (sg == 1 && mt == 4) return fused_t<1, 4>(c, p, xhat, w, y, r, y0, s, chained, em);
  if (sg == 2 && mt == 1) return fused_t<2, 1>(c, p, xhat, w, y, r, y0, s, chained, em);
  if (sg == 2 && mt == 2) return fused_t<2, 2>(c, p, xhat, w, y, r, y0, s, chained, em);
  return cudaErrorInvalidValue;
}

cudaError_t launch_pack_weights(const DevConsts& c, const PlanDev& p, const uint64_t* kernel, void* w,
                                cudaStream_t s) {
  const size_t N = 1ull << c.log_n;
  const size_t wb = c.word_bits / 8;
  cudaError_t e = cudaMemsetAsync(w, 0, (size_t)p.M * p.G * c.L * N * wb, s);
  if (e != cudaSuccess) return e;
  const size_t total = (size_t)p.M * p.C * p.kh0 * p.kw0;
  if (!total) return cudaGetLastError();
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (c.word_bits == 64)
    k_pack_weights<uint64_t><<<blocks, 256, 0, s>>>(kernel, static_cast<uint64_t*>(w), c, p);
  else
    k_pack_weights<uint32_t><<<blocks, 256, 0, s>>>(kernel, static_cast<uint32_t*>(w), c, p);
  return cudaGetLastError();
}

cudaError_t launch_pack_fc_weights(const DevConsts& c, const PlanDev& p, const uint64_t* Wm, void* w, cudaStream_t s) {
  const size_t N = 1ull << c.log_n;
  const size_t wb = c.word_bits / 8;
  cudaError_t e = cudaMemsetAsync(w, 0, (size_t)p.M * p.G * c.L * N * wb, s);
  if (e != cudaSuccess) return e;
  const size_t total = (size_t)p.no * p.C;
  if (!total) return cudaGetLastError();
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (c.word_bits == 64)
    k_pack_fc_weights<uint64_t><<<blocks, 256, 0, s>>>(Wm, static_cast<uint64_t*>(w), c, p);
  else
    k_pack_fc_weights<uint32_t><<<blocks, 256, 0, s>>>(Wm, static_cast<uint32_t*>(w), c, p);
  return cudaGetLastError();
}

cudaError_t launch_ntt_inv_tail_lwe(const DevConsts& c, const MsConsts& ms, const void* polys, size_t n_ct,
                                    const uint64_t* r, void* a_out, void* b_out, uint64_t* y0, const PlanDev& pl,
                                    cudaStream_t s, bool chained, const void* em) {
  if (n_ct == 0) return cudaSuccess;
  if (c.log_n != 12 || 4 * n_ct > 0x7fffffffull) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)(4 * n_ct)), block(LWE_G * c.L);  // (ct, component, half) x limbs
  const int nd = (int)(c.L - ms.Lk);
#define SECN_LWE(AR, WT, ND)                                                                                   \
  return launch_pdl(c, k_ntt_inv_tail_lwe<AR, ND>, grid, block, 0, s, static_cast<const WT*>(polys), c, ms, r, \
                    static_cast<WT*>(a_out), static_cast<WT*>(b_out), y0, pl, chained ? 1 : 0, static_cast<const WT*>(em))
  if (c.word_bits == 64) {
    if (nd == 1) SECN_LWE(Arith64, uint64_t, 1);  // 64-bit limbs: one dropped prime (P < 2^62)
  } else {
    if (nd == 1) SECN_LWE(Arith32, uint32_t, 1);
    if (nd == 2) SECN_LWE(Arith32, uint32_t, 2);
  }
#undef SECN_LWE
  return cudaErrorInvalidValue;
}

cudaError_t launch_enc_add(const DevConsts& c, void* ct, const uint64_t* v, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const size_t total = n * c.L * (1ull << c.log_n);
  const size_t blocks = (total + 255) / 256;
  const size_t cap = (size_t)c.tune.num_sms * 32;
  const unsigned b = (unsigned)(blocks < cap ? blocks : cap);
  if (c.word_bits == 64)
    k_enc_add<Arith64><<<b, 256, 0, s>>>(static_cast<uint64_t*>(ct), v, c, n);
  else
    k_enc_add<Arith32><<<b, 256, 0, s>>>(static_cast<uint32_t*>(ct), v, c, n);
  return cudaGetLastError();
}

cudaError_t launch_extract_share(const DevConsts& c, const PlanDev& p, const uint64_t* r, uint64_t* y0,
                                 cudaStream_t s) {
  const size_t total = (size_t)p.M * p.OH * p.OW;
  if (total) {
    cudaError_t e = launch_pdl(c, k_extract_share, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, r, y0, c, p);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_mask_draw(const DevConsts& c, const MaskGen& g, size_t n_ct, uint64_t* r, cudaStream_t s) {
  if (n_ct == 0) return cudaSuccess;
  const size_t half = (size_t)1 << (c.log_n - 1), pairs = n_ct * half;
  const size_t blocks = (pairs + 255) / 256, cap = (size_t)c.tune.num_sms * 16;
  return launch_pdl(c, k_mask_draw, dim3((unsigned)(blocks < cap ? blocks : cap)), dim3(256), 0, s, r, g, pairs,
                    (uint32_t)half, c.t_bits);
}

cudaError_t launch_mask_encode(const DevConsts& c, const PlanDev& p, size_t n_act, const uint64_t* r, const MaskGen& g,
                               void* em, uint64_t* y0, cudaStream_t s, bool chained) {
  if (n_act == 0) return cudaSuccess;
  if (n_act > 65535) return cudaErrorInvalidValue;  // grid.y
  const dim3 grid((unsigned)(((1u << c.log_n) / MASK_COEFS + 255) / 256), (unsigned)n_act);
  if (c.word_bits == 64)
    return launch_pdl(c, k_mask_encode<Arith64>, grid, dim3(256), 0, s, static_cast<uint64_t*>(em), y0, r, g, c, p,
                      (uint32_t)n_act, chained ? 0 : 1);
  return launch_pdl(c, k_mask_encode<Arith32>, grid, dim3(256), 0, s, static_cast<uint32_t*>(em), y0, r, g, c, p,
                    (uint32_t)n_act, chained ? 0 : 1);
}

cudaError_t launch_check_range(const DevConsts& c, const void* v, size_t n_words, int kind, uint32_t* flag,
                               cudaStream_t s) {
  if (n_words == 0) return cudaSuccess;
  const size_t blocks = (n_words + 255) / 256;
  const size_t cap = (size_t)c.tune.num_sms * 16;
  const unsigned b = (unsigned)(blocks < cap ? blocks : cap);
  if (kind == 0 && c.word_bits == 32)
    k_check_range<uint32_t><<<b, 256, 0, s>>>(static_cast<const uint32_t*>(v), n_words, c, kind, flag);
  else
    k_check_range<uint64_t><<<b, 256, 0, s>>>(static_cast<const uint64_t*>(v), n_words, c, kind, flag);
  return cudaGetLastError();
}

}  // namespace secn

#ifdef SECN_PROBE
extern "C" int secn_probe_read(unsigned long long* dst, size_t n) {
  return cudaMemcpyFromSymbol(dst, secn::g_probe, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -5;
}
extern "C" int secn_probe_clear(void) {
  static unsigned long long z[65536 * 2 + 64];
  return cudaMemcpyToSymbol(secn::g_probe, z, sizeof(z)) == cudaSuccess ? 0 : -5;
}
#endif
