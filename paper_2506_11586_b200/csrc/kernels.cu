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

#include "internal.h"
#include "modarith.cuh"
#include "ntt_core.cuh"

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
};
template <>
struct Tab<Arith32> {
  __device__ static const uint2* fwd(const DevConsts& c) { return c.tw32_fwd; }
  __device__ static const uint2* inv(const DevConsts& c) { return c.tw32_inv; }
  __device__ static uint2 pair(uint64_t w, uint64_t wp) { return make_uint2((uint32_t)w, (uint32_t)wp); }
};

// enc_j(v) = round(Q v / t) mod q_j (reading R2) = floor(Q/t) v + floor(((Q mod t) v + t/2) / t),
// canonical in [0, q), with 64-bit arithmetic (any q < 2^61, v < 2^44).
__device__ __forceinline__ uint64_t enc_mod(uint64_t v, int j, const DevConsts& c) {
  const uint64_t q = c.q[j];
  const uint64_t a = shoup(v, c.delta[j], c.delta_p[j], q);  // [0, 2q)
  uint64_t lo = c.qmt * v, hi = mulhi(c.qmt, v);
  const uint64_t half = 1ull << (c.t_bits - 1);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(half));
  const uint64_t frac = (hi << (64 - c.t_bits)) | (lo >> c.t_bits);  // < Q mod t < 2^t_bits
  const uint64_t b = frac - mulhi(frac, c.one_p[j]) * q;              // [0, 2q)
  return csub(csub(a + b, 2 * q), q);
}

template <int LOGN>
constexpr int ntt_min_blocks() { return LOGN == 12 ? 3 : 1; }

// ------------------------------------------------------------------------------------------
// K1: forward NTT of limb-polys [P][N] (limb j = p mod L), optionally fused server-share add
// on the b component of ciphertexts [n][2][L][N]: b_j += enc_j(x0[n]). The
// first radix-16 round reads global memory directly (its tasks are coalesced).
template <class A, int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16, ntt_min_blocks<LOGN>())
    k_ntt_fwd(const typename A::W* in, typename A::W* out, const __grid_constant__ DevConsts c,
              const uint64_t* __restrict__ x0) {
  using W = typename A::W;
  using R0 = CtRound<LOGN, 0>;
  constexpr int N = 1 << LOGN, T = N / 16;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const size_t p = blockIdx.x;
  const int j = (int)(p % c.L);
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::fwd(c) + (size_t)j * N;
  const W* src = in + p * N;
  const bool share = x0 != nullptr && ((p / c.L) & 1);
  const uint64_t* xs = share ? x0 + (p / (2 * c.L)) * N : nullptr;
  W x[16];
#pragma unroll
  for (int k = 0; k < R0::NT; ++k)
#pragma unroll
    for (int i = 0; i < R0::GK; ++i) {
      const uint32_t e = R0::addr(k, i);
      W v = src[e];
      if (share) v += (W)enc_mod(__ldg(&xs[e]), j, c);  // < 2q: inside the CT domain
      x[k * R0::GK + i] = v;
    }
  ct_compute<A, LOGN, 0>(x, tw, q, qb);
  ct_store<A, LOGN, 0>(x, sm);
  __syncthreads();
  ct_rounds_smem<A, LOGN, R0::K>(sm, tw, q, qb);
  W* dst = out + p * N;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    dst[e] = A::canon_ct(sm[swz(e)], q);
  }
}

// K3 (+A7 fused): inverse NTT of limb-polys in place; if r != NULL, on the b component of
// ciphertexts [n][2][L][N]: b_j += enc_j(r[n]) after the transform. The last
// radix-16 round writes global memory directly (its tasks are coalesced).
template <class A, int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16, ntt_min_blocks<LOGN>())
    k_ntt_inv(typename A::W* polys, const __grid_constant__ DevConsts c, const uint64_t* __restrict__ r) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN, T = N / 16;
  constexpr int LL = GsLast<LOGN>::value;
  using RL = GsRound<LOGN, LL>;
  extern __shared__ __align__(16) unsigned char smraw[];
  W* sm = reinterpret_cast<W*>(smraw);
  const size_t p = blockIdx.x;
  const int j = (int)(p % c.L);
  const W q = (W)c.q[j], qb = A::bound(q);
  const typename A::Tw* tw = Tab<A>::inv(c) + (size_t)j * N;
  const typename A::Tw ninv = Tab<A>::pair(c.ninv[j], c.ninv_p[j]);
  const typename A::Tw wl = Tab<A>::pair(c.wlast[j], c.wlast_p[j]);
  W* buf = polys + p * N;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    sm[swz(e)] = buf[e];
  }
  __syncthreads();
  gs_rounds_smem_but_last<A, LOGN, 0>(sm, tw, q, qb, ninv, wl);
  W x[16];
  gs_load<A, LOGN, LL>(x, sm);
  gs_compute<A, LOGN, LL>(x, tw, q, qb, ninv, wl);
  const bool mask = r != nullptr && ((p / c.L) & 1);
  const uint64_t* rs = mask ? r + (p / (2 * c.L)) * N : nullptr;
#pragma unroll
  for (int k = 0; k < RL::NT; ++k)
#pragma unroll
    for (int i = 0; i < RL::GK; ++i) {
      const uint32_t e = RL::addr(k, i);
      W v = A::canon_gs(x[k * RL::GK + i], q);
      if (mask) {
        v += (W)enc_mod(__ldg(&rs[e]), j, c);  // < 2q
        v = v >= q ? v - q : v;
      }
      buf[e] = v;
    }
}

// ------------------------------------------------------------------------------------------
// A4: NTT-domain multiply-accumulate ("performs all HE MAC operations in NTT"):
//   Y^[m,s,c,j,e] = sum_g X^[g,s,c,j,e] * W[m,g,j,e] mod q_j
// Per coefficient e this is a small (M x G) . (G x 2S) matrix product. A CTA owns 256
// coefficients of limb j (one per thread), a tile of output channels and a group of SG spatial
// blocks (both ciphertext components). The thread's X^ values are staged once and reused for
// every m of the tile, so the weights stream from HBM exactly once; each thread keeps the
// weight row W[m+1, :, j, e] in flight in registers while it multiplies row m. Products
// accumulate lazily (128-bit for 64-bit words, 64-bit for 32-bit words) with one reduction per
// output word.
constexpr int MAC_THREADS = 256;

// 64-bit words: X^ staged in shared memory ([G][2*SG][256] thread-private columns).
template <int SG, int GMAX>
__global__ void __launch_bounds__(MAC_THREADS, GMAX <= 16 ? 2 : 1)
    k_mac64(const uint64_t* __restrict__ xhat, const uint64_t* __restrict__ w, uint64_t* __restrict__ y,
            const __grid_constant__ DevConsts c, PlanDev pl, int m_tile, int n_mtiles) {
  extern __shared__ uint64_t xs[];
  const int N = 1 << c.log_n, L = c.L, G = pl.G, S = pl.S;
  const int j = blockIdx.y;
  const uint32_t e = blockIdx.x * MAC_THREADS + threadIdx.x;
  const int mt = blockIdx.z % n_mtiles, sgi = blockIdx.z / n_mtiles;
  const int s0 = sgi * SG;
  const int ns = min(SG, S - s0);
  const uint64_t q = c.q[j], r64 = c.r64[j], r64p = c.r64_p[j], onep = c.one_p[j];
  for (int g = 0; g < G; ++g)
    for (int a = 0; a < 2 * ns; ++a)
      xs[(g * 2 * SG + a) * MAC_THREADS + threadIdx.x] =
          xhat[((((size_t)g * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e];
  const int m_begin = mt * m_tile, m_end = min((int)pl.M, m_begin + m_tile);
  const size_t gstride = (size_t)L * N, mstride = (size_t)G * L * N;
  const uint64_t* wp = w + ((size_t)m_begin * G * L + j) * N + e;
  uint64_t wr[GMAX];
#pragma unroll
  for (int g = 0; g < GMAX; ++g)
    if (g < G) wr[g] = __ldg(wp + g * gstride);
  for (int m = m_begin; m < m_end; ++m) {
    const bool more = m + 1 < m_end;
    const uint64_t* wn = wp + (size_t)(m + 1 - m_begin) * mstride;
    uint64_t lo[2 * SG], hi[2 * SG];
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a) lo[a] = hi[a] = 0;
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < G) {
        const uint64_t wc = wr[g];
        if (more) wr[g] = __ldg(wn + g * gstride);
#pragma unroll
        for (int a = 0; a < 2 * SG; ++a)
          if (a < 2 * ns) mac128(lo[a], hi[a], xs[(g * 2 * SG + a) * MAC_THREADS + threadIdx.x], wc);
        if (g % 62 == 61) {  // keep the 128-bit sums below 2^128 (q < 2^61)
#pragma unroll
          for (int a = 0; a < 2 * SG; ++a) {
            lo[a] = reduce128(lo[a], hi[a], q, r64, r64p, onep);
            hi[a] = 0;
          }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a)
      if (a < 2 * ns)
        y[((((size_t)m * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e] = reduce128(lo[a], hi[a], q, r64, r64p, onep);
  }
}

// 32-bit words: X^ held in registers ([GMAX][2*SG] words per thread), products summed exactly
// in 64 bits (32-bit contexts require q < 2^28, so each product is < 2^56 and any G <= 256
// fits), one IMAD.WIDE per MAC.
__device__ __forceinline__ uint32_t reduce64(uint64_t a, uint64_t q, uint64_t onep) {
  const uint64_t r = a - mulhi(a, onep) * q;  // [0, 2q)
  return (uint32_t)(r >= q ? r - q : r);
}

template <int SG, int GMAX>
__global__ void __launch_bounds__(MAC_THREADS, GMAX <= 16 ? 2 : 1)
    k_mac32(const uint32_t* __restrict__ xhat, const uint32_t* __restrict__ w, uint32_t* __restrict__ y,
            const __grid_constant__ DevConsts c, PlanDev pl, int m_tile, int n_mtiles) {
  const int N = 1 << c.log_n, L = c.L, G = pl.G, S = pl.S;
  const int j = blockIdx.y;
  const uint32_t e = blockIdx.x * MAC_THREADS + threadIdx.x;
  const int mt = blockIdx.z % n_mtiles, sgi = blockIdx.z / n_mtiles;
  const int s0 = sgi * SG;
  const int ns = min(SG, S - s0);
  const uint64_t q = c.q[j], onep = c.one_p[j];
  uint32_t xr[GMAX][2 * SG];
#pragma unroll
  for (int g = 0; g < GMAX; ++g)
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a)
      xr[g][a] = (g < G && a < 2 * ns) ? xhat[((((size_t)g * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e] : 0u;
  const int m_begin = mt * m_tile, m_end = min((int)pl.M, m_begin + m_tile);
  const size_t gstride = (size_t)L * N, mstride = (size_t)G * L * N;
  const uint32_t* wp = w + ((size_t)m_begin * G * L + j) * N + e;
  uint32_t wr[GMAX];
#pragma unroll
  for (int g = 0; g < GMAX; ++g)
    if (g < G) wr[g] = __ldg(wp + g * gstride);
  for (int m = m_begin; m < m_end; ++m) {
    const bool more = m + 1 < m_end;
    const uint32_t* wn = wp + (size_t)(m + 1 - m_begin) * mstride;
    uint64_t acc[2 * SG];
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a) acc[a] = 0;
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g < G) {
        const uint32_t wc = wr[g];
        if (more) wr[g] = __ldg(wn + g * gstride);
#pragma unroll
        for (int a = 0; a < 2 * SG; ++a) acc[a] += (uint64_t)xr[g][a] * wc;
      }
    }
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a)
      if (a < 2 * ns) y[((((size_t)m * S + s0 + (a >> 1)) * 2 + (a & 1)) * L + j) * N + e] = reduce64(acc[a], q, onep);
  }
}

// ------------------------------------------------------------------------------------------
// A3 packing: kernel [M][C][kh][kw] (< 2^t) -> mirrored coefficient-domain polys
// w[m][g][j][O - c*Hw*Ww - l*Ww - l'] = lift_j(K[m, g*Cw+c, l, l']) (reading R3: centred lift).
// The target must be zero-filled before.
template <class W>
__global__ void k_pack_weights(const uint64_t* __restrict__ kern, W* __restrict__ w,
                               const __grid_constant__ DevConsts c, PlanDev pl) {
  const size_t total = (size_t)pl.M * pl.C * pl.kh * pl.kw;
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint32_t l2 = idx % pl.kw;
  const uint32_t l = (idx / pl.kw) % pl.kh;
  const uint32_t ch = (idx / ((size_t)pl.kw * pl.kh)) % pl.C;
  const uint32_t m = idx / ((size_t)pl.kw * pl.kh * pl.C);
  const uint32_t g = ch / pl.Cw, cc = ch % pl.Cw;
  const uint32_t coef = pl.O - cc * pl.Hw * pl.Ww - l * pl.Ww - l2;
  const uint64_t t = 1ull << c.t_bits;
  const uint64_t v = kern[idx] & (t - 1);
  const size_t N = 1ull << c.log_n;
  for (uint32_t j = 0; j < c.L; ++j) {
    const uint64_t q = c.q[j];
    const uint64_t lifted = v >= t / 2 ? (q - (t - v) % q) % q : v % q;
    w[(((size_t)m * pl.G + g) * c.L + j) * N + coef] = (W)lifted;
  }
}

// A6 / A7 standalone: ct [n][2][L][N], b_j += enc_j(v[n][N]).
template <class W>
__global__ void k_enc_add(W* __restrict__ ct, const uint64_t* __restrict__ v, const __grid_constant__ DevConsts c,
                          size_t n) {
  const size_t N = 1ull << c.log_n;
  const size_t total = n * c.L * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t e = idx % N;
    const uint32_t j = (idx / N) % c.L;
    const size_t i = idx / (N * c.L);
    W* b = ct + ((i * 2 + 1) * c.L + j) * N + e;
    const uint64_t q = c.q[j];
    const uint64_t s = (uint64_t)*b + enc_mod(v[i * N + e], j, c);  // [0, 2q)
    *b = (W)(s >= q ? s - q : s);
  }
}

// Designated server share y0[m][oy][ox] = (t - r[m*S+s][O + i*Ww + j]) mod t.
__global__ void k_extract_share(const uint64_t* __restrict__ r, uint64_t* __restrict__ y0,
                                const __grid_constant__ DevConsts c, PlanDev pl) {
  const size_t total = (size_t)pl.M * pl.OH * pl.OW;
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const uint32_t ox = idx % pl.OW, oy = (idx / pl.OW) % pl.OH, m = idx / ((size_t)pl.OW * pl.OH);
  const uint32_t py = oy * pl.sh, px = ox * pl.sh;
  const uint32_t bh = py / (pl.Hw - pl.kh + 1), i = py % (pl.Hw - pl.kh + 1);
  const uint32_t bw = px / (pl.Ww - pl.kw + 1), jj = px % (pl.Ww - pl.kw + 1);
  const uint32_t s = bh * pl.nbw + bw;
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

template <class A, int LOGN>
static cudaError_t ntt_fwd_t(const DevConsts& c, const void* in, void* out, size_t P, const uint64_t* x0,
                             cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  const size_t smem = N * sizeof(W);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ntt_fwd<A, LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (size_t off = 0; off < P; off += 0x7fffffff) {
    const size_t cnt = P - off < 0x7fffffff ? P - off : 0x7fffffff;
    k_ntt_fwd<A, LOGN><<<(unsigned)cnt, N / 16, smem, s>>>(static_cast<const W*>(in) + off * N,
                                                          static_cast<W*>(out) + off * N, c, x0);
  }
  return cudaGetLastError();
}

template <class A, int LOGN>
static cudaError_t ntt_inv_t(const DevConsts& c, void* polys, size_t P, const uint64_t* r, cudaStream_t s) {
  using W = typename A::W;
  constexpr int N = 1 << LOGN;
  const size_t smem = N * sizeof(W);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ntt_inv<A, LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (size_t off = 0; off < P; off += 0x7fffffff) {
    const size_t cnt = P - off < 0x7fffffff ? P - off : 0x7fffffff;
    k_ntt_inv<A, LOGN><<<(unsigned)cnt, N / 16, smem, s>>>(static_cast<W*>(polys) + off * N, c, r);
  }
  return cudaGetLastError();
}

cudaError_t launch_ntt_fwd(const DevConsts& c, const void* in, void* out, size_t P, const uint64_t* x0,
                           cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  if (c.word_bits == 64) {
    switch (c.log_n) {
      case 12: return ntt_fwd_t<Arith64, 12>(c, in, out, P, x0, s);
      case 13: return ntt_fwd_t<Arith64, 13>(c, in, out, P, x0, s);
      case 14: return ntt_fwd_t<Arith64, 14>(c, in, out, P, x0, s);
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

cudaError_t launch_ntt_inv(const DevConsts& c, void* polys, size_t P, const uint64_t* r, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  if (c.word_bits == 64) {
    switch (c.log_n) {
      case 12: return ntt_inv_t<Arith64, 12>(c, polys, P, r, s);
      case 13: return ntt_inv_t<Arith64, 13>(c, polys, P, r, s);
      case 14: return ntt_inv_t<Arith64, 14>(c, polys, P, r, s);
    }
  } else {
    switch (c.log_n) {
      case 12: return ntt_inv_t<Arith32, 12>(c, polys, P, r, s);
      case 13: return ntt_inv_t<Arith32, 13>(c, polys, P, r, s);
      case 14: return ntt_inv_t<Arith32, 14>(c, polys, P, r, s);
    }
  }
  return cudaErrorInvalidValue;
}

// m-tile: about 4 waves of 2 CTAs per SM, at least 8 channels per CTA to amortise the X^ staging
static int mac_m_tile(const DevConsts& c, const PlanDev& p, int n_sg) {
  const long ctas_no_m = (long)((1 << c.log_n) / MAC_THREADS) * c.L * n_sg;
  int m_tile = (int)(((long)p.M * ctas_no_m + 1183) / 1184);
  if (m_tile < 8) m_tile = 8;
  if (m_tile > (int)p.M) m_tile = p.M;
  return m_tile;
}

template <int SG, int GMAX>
static cudaError_t mac64_t(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                           cudaStream_t s) {
  const int N = 1 << c.log_n;
  const size_t smem = (size_t)p.G * 2 * SG * MAC_THREADS * sizeof(uint64_t);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_mac64<SG, GMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int n_sg = (p.S + SG - 1) / SG;
  const int m_tile = mac_m_tile(c, p, n_sg);
  const int n_mtiles = (p.M + m_tile - 1) / m_tile;
  dim3 grid(N / MAC_THREADS, c.L, n_mtiles * n_sg);
  k_mac64<SG, GMAX><<<grid, MAC_THREADS, smem, s>>>(static_cast<const uint64_t*>(xhat), static_cast<const uint64_t*>(w),
                                                    static_cast<uint64_t*>(y), c, p, m_tile, n_mtiles);
  return cudaGetLastError();
}

template <int GMAX>
static cudaError_t mac64_g(int sg, const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                           cudaStream_t s) {
  switch (sg) {
    case 1: return mac64_t<1, GMAX>(c, p, xhat, w, y, s);
    case 2: return mac64_t<2, GMAX>(c, p, xhat, w, y, s);
    case 3: return mac64_t<3, GMAX>(c, p, xhat, w, y, s);
    default: return mac64_t<4, GMAX>(c, p, xhat, w, y, s);
  }
}

template <int SG, int GMAX>
static cudaError_t mac32_t(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                           cudaStream_t s) {
  const int N = 1 << c.log_n;
  const int n_sg = (p.S + SG - 1) / SG;
  const int m_tile = mac_m_tile(c, p, n_sg);
  const int n_mtiles = (p.M + m_tile - 1) / m_tile;
  dim3 grid(N / MAC_THREADS, c.L, n_mtiles * n_sg);
  k_mac32<SG, GMAX><<<grid, MAC_THREADS, 0, s>>>(static_cast<const uint32_t*>(xhat), static_cast<const uint32_t*>(w),
                                                 static_cast<uint32_t*>(y), c, p, m_tile, n_mtiles);
  return cudaGetLastError();
}

template <int GMAX>
static cudaError_t mac32_g(int sg, const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                           cudaStream_t s) {
  // X^ registers: GMAX * 2 * SG <= 48 words per thread (no spills at 128 registers)
  constexpr int SGMAX = GMAX >= 16 ? 1 : (24 / GMAX < 4 ? 24 / GMAX : 4);
  if (sg > SGMAX) sg = SGMAX;
  switch (sg) {
    case 1: return mac32_t<1, GMAX>(c, p, xhat, w, y, s);
    case 2: return mac32_t<(SGMAX >= 2 ? 2 : 1), GMAX>(c, p, xhat, w, y, s);
    case 3: return mac32_t<(SGMAX >= 3 ? 3 : 1), GMAX>(c, p, xhat, w, y, s);
    default: return mac32_t<SGMAX, GMAX>(c, p, xhat, w, y, s);
  }
}

cudaError_t launch_mac(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                       cudaStream_t s) {
  if (p.M == 0 || p.S == 0) return cudaSuccess;
  if (c.word_bits == 64) {
    // s-group: as many spatial blocks (<= 4) as keep the X^ tile within 100 KiB (2 CTAs / SM)
    const size_t per_s = (size_t)p.G * 2 * MAC_THREADS * sizeof(uint64_t);
    if (per_s > 200 * 1024) return cudaErrorInvalidValue;  // G > 50
    int sg = 4;
    while (sg > 1 && per_s * sg > 100 * 1024) --sg;
    if (sg > (int)p.S) sg = p.S;
    if (p.G <= 8) return mac64_g<8>(sg, c, p, xhat, w, y, s);
    if (p.G <= 16) return mac64_g<16>(sg, c, p, xhat, w, y, s);
    if (p.G <= 32) return mac64_g<32>(sg < 2 ? sg : 2, c, p, xhat, w, y, s);
    return mac64_g<64>(1, c, p, xhat, w, y, s);
  }
  if (p.G > 32) return cudaErrorInvalidValue;
  const int sg = p.S < 4 ? (int)p.S : 4;
  if (p.G <= 4) return mac32_g<4>(sg, c, p, xhat, w, y, s);
  if (p.G <= 8) return mac32_g<8>(sg, c, p, xhat, w, y, s);
  if (p.G <= 16) return mac32_g<16>(sg, c, p, xhat, w, y, s);
  return mac32_g<32>(sg, c, p, xhat, w, y, s);
}

cudaError_t launch_pack_weights(const DevConsts& c, const PlanDev& p, const uint64_t* kernel, void* w,
                                cudaStream_t s) {
  const size_t N = 1ull << c.log_n;
  const size_t wb = c.word_bits / 8;
  cudaError_t e = cudaMemsetAsync(w, 0, (size_t)p.M * p.G * c.L * N * wb, s);
  if (e != cudaSuccess) return e;
  const size_t total = (size_t)p.M * p.C * p.kh * p.kw;
  if (!total) return cudaGetLastError();
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (c.word_bits == 64)
    k_pack_weights<uint64_t><<<blocks, 256, 0, s>>>(kernel, static_cast<uint64_t*>(w), c, p);
  else
    k_pack_weights<uint32_t><<<blocks, 256, 0, s>>>(kernel, static_cast<uint32_t*>(w), c, p);
  return cudaGetLastError();
}

cudaError_t launch_enc_add(const DevConsts& c, void* ct, const uint64_t* v, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const size_t total = n * c.L * (1ull << c.log_n);
  const size_t blocks = (total + 255) / 256;
  const unsigned b = (unsigned)(blocks < 148 * 32 ? blocks : 148 * 32);
  if (c.word_bits == 64)
    k_enc_add<uint64_t><<<b, 256, 0, s>>>(static_cast<uint64_t*>(ct), v, c, n);
  else
    k_enc_add<uint32_t><<<b, 256, 0, s>>>(static_cast<uint32_t*>(ct), v, c, n);
  return cudaGetLastError();
}

cudaError_t launch_extract_share(const DevConsts& c, const PlanDev& p, const uint64_t* r, uint64_t* y0,
                                 cudaStream_t s) {
  const size_t total = (size_t)p.M * p.OH * p.OW;
  if (total) k_extract_share<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(r, y0, c, p);
  return cudaGetLastError();
}

cudaError_t launch_check_range(const DevConsts& c, const void* v, size_t n_words, int kind, uint32_t* flag,
                               cudaStream_t s) {
  if (n_words == 0) return cudaSuccess;
  const size_t blocks = (n_words + 255) / 256;
  const unsigned b = (unsigned)(blocks < 148 * 16 ? blocks : 148 * 16);
  if (kind == 0 && c.word_bits == 32)
    k_check_range<uint32_t><<<b, 256, 0, s>>>(static_cast<const uint32_t*>(v), n_words, c, kind, flag);
  else
    k_check_range<uint64_t><<<b, 256, 0, s>>>(static_cast<const uint64_t*>(v), n_words, c, kind, flag);
  return cudaGetLastError();
}

}  // namespace secn
