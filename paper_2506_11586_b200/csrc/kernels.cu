// libsecn device kernels for sm_100a: RNS negacyclic NTT/INTT (64-bit Shoup, Harvey lazy
// butterflies, shared-memory radix-16 rounds), fused share-add / mask-add, the NTT-domain
// ct x pt multiply-accumulate, weight packing, and the designated-share gather.
//
// Paper: PAPER.md:376-380 (§6.2 NTT preprocessing: "transforms each ciphertext with NTT,
// performs all HE MAC operations in NTT, and only transforms the final HE results back"),
// PAPER.md:431 (§7: server share add, random mask), PAPER.md:668-679 (App. C.1 NTT).
#include <cstdio>

#include "internal.h"
#include "modarith.cuh"

namespace secn {

// ------------------------------------------------------------------------------------------
// shared-memory layout of one limb-poly: 64-bit words, XOR swizzle of the low 4 index bits
// with bits 4..7 -- conflict-free (16 distinct banks pairs per half-warp) for every
// radix-16 round pattern below and for contiguous copies (checked by tools/banks.py).
__device__ __forceinline__ uint32_t swz(uint32_t e) { return e ^ ((e >> 4) & 15u); }

// enc_j(v) = round(Q v / t) mod q_j (reading R2) = floor(Q/t) v + floor(((Q mod t) v + t/2) / t),
// returned lazily in [0, 3q).
__device__ __forceinline__ uint64_t enc_lazy(uint64_t v, int j, const DevConsts& c) {
  const uint64_t a = shoup(v, c.delta[j], c.delta_p[j], c.q[j]);  // [0, 2q)
  uint64_t lo = c.qmt * v, hi = mulhi(c.qmt, v);
  const uint64_t half = 1ull << (c.t_bits - 1);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(half));
  const uint64_t frac = (hi << (64 - c.t_bits)) | (lo >> c.t_bits);  // < Q mod t < 2^t_bits < q
  return a + frac;
}

// ------------------------------------------------------------------------------------------
// Cooley-Tukey round: stages s0 .. s0+K-1 of the forward transform
//   for stage s (m = 2^s groups, half-distance t = N/2^(s+1)): group i uses psi^brv(m+i).
// A task is the 2^K elements blk*B + off + i*D (B = N >> s0, D = B >> K) that interact in
// these K stages; each thread owns 16/2^K tasks, i.e. 16 words in registers.
template <int LOGN, int K>
__device__ __forceinline__ void ct_round(uint64_t* sm, int s0, const ulonglong2* __restrict__ tw, uint64_t q,
                                         uint64_t q2) {
  constexpr int T = (1 << LOGN) / 16;
  constexpr int GK = 1 << K, NT = 16 / GK;
  const int logB = LOGN - s0, logD = logB - K;
  const int tid = threadIdx.x;
  uint64_t x[16];
  uint32_t base[NT], blk[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const uint32_t tau = tid + k * T;
    blk[k] = tau >> logD;
    base[k] = (blk[k] << logB) + (tau & ((1u << logD) - 1));
#pragma unroll
    for (int i = 0; i < GK; ++i) x[k * GK + i] = sm[swz(base[k] + (i << logD))];
  }
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int half = GK >> (p + 1);
#pragma unroll
    for (int k = 0; k < NT; ++k) {
#pragma unroll
      for (int u = 0; u < (1 << p); ++u) {
        const ulonglong2 w = __ldg(&tw[(1u << (s0 + p)) + (blk[k] << p) + u]);
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const int a = k * GK + u * (GK >> p) + i;
          ct_bfly(x[a], x[a + half], w.x, w.y, q, q2);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NT; ++k)
#pragma unroll
    for (int i = 0; i < GK; ++i) sm[swz(base[k] + (i << logD))] = x[k * GK + i];
}

// Gentleman-Sande round: levels l0 .. l0+K-1 of the inverse transform
//   level l (half-distance t = 2^l, h = N/2^(l+1) groups): group i uses psi^-brv(h+i).
// The final level (h = 1) folds N^-1: X' = (U+V) N^-1, Y' = (U-V) psi^-brv(1) N^-1.
template <int LOGN, int K>
__device__ __forceinline__ void gs_round(uint64_t* sm, int l0, const ulonglong2* __restrict__ tw, uint64_t q,
                                         uint64_t q2, uint64_t ninv, uint64_t ninvp, uint64_t wl, uint64_t wlp) {
  constexpr int T = (1 << LOGN) / 16;
  constexpr int GK = 1 << K, NT = 16 / GK;
  const int logB = l0 + K, logD = l0;
  const int tid = threadIdx.x;
  uint64_t x[16];
  uint32_t base[NT], blk[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    const uint32_t tau = tid + k * T;
    blk[k] = tau >> logD;
    base[k] = (blk[k] << logB) + (tau & ((1u << logD) - 1));
#pragma unroll
    for (int i = 0; i < GK; ++i) x[k * GK + i] = sm[swz(base[k] + (i << logD))];
  }
#pragma unroll
  for (int p = 0; p < K; ++p) {
    const int dist = 1 << p;
    const int lvl = l0 + p;
    if (lvl == LOGN - 1) {  // last level: single group, N^-1 folded in
#pragma unroll
      for (int k = 0; k < NT; ++k)
#pragma unroll
        for (int i = 0; i < GK; ++i) {
          if (i & dist) continue;
          const uint64_t u = x[k * GK + i], v = x[k * GK + i + dist];
          x[k * GK + i] = shoup(u + v, ninv, ninvp, q);
          x[k * GK + i + dist] = shoup(u - v + q2, wl, wlp, q);
        }
    } else {
      const uint32_t h = (1u << LOGN) >> (lvl + 1);
#pragma unroll
      for (int k = 0; k < NT; ++k) {
#pragma unroll
        for (int gi = 0; gi < (GK >> (p + 1)); ++gi) {
          const ulonglong2 w = __ldg(&tw[h + (blk[k] << (K - p - 1)) + gi]);
#pragma unroll
          for (int i = 0; i < dist; ++i) {
            const int a = k * GK + gi * (2 * dist) + i;
            gs_bfly(x[a], x[a + dist], w.x, w.y, q, q2);
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NT; ++k)
#pragma unroll
    for (int i = 0; i < GK; ++i) sm[swz(base[k] + (i << logD))] = x[k * GK + i];
}

template <int LOGN>
__device__ __forceinline__ void ntt_fwd_smem(uint64_t* sm, const ulonglong2* tw, uint64_t q, uint64_t q2) {
  ct_round<LOGN, 4>(sm, 0, tw, q, q2);
  __syncthreads();
  ct_round<LOGN, 4>(sm, 4, tw, q, q2);
  __syncthreads();
  ct_round<LOGN, 4>(sm, 8, tw, q, q2);
  __syncthreads();
  if constexpr (LOGN > 12) {
    ct_round<LOGN, LOGN - 12>(sm, 12, tw, q, q2);
    __syncthreads();
  }
}

template <int LOGN>
__device__ __forceinline__ void ntt_inv_smem(uint64_t* sm, const ulonglong2* tw, uint64_t q, uint64_t q2,
                                             uint64_t ninv, uint64_t ninvp, uint64_t wl, uint64_t wlp) {
  gs_round<LOGN, 4>(sm, 0, tw, q, q2, ninv, ninvp, wl, wlp);
  __syncthreads();
  gs_round<LOGN, 4>(sm, 4, tw, q, q2, ninv, ninvp, wl, wlp);
  __syncthreads();
  gs_round<LOGN, 4>(sm, 8, tw, q, q2, ninv, ninvp, wl, wlp);
  __syncthreads();
  if constexpr (LOGN > 12) {
    gs_round<LOGN, LOGN - 12>(sm, 12, tw, q, q2, ninv, ninvp, wl, wlp);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------
// K1: forward NTT of limb-polys [P][N] (limb j = p mod L), optionally fused server-share add
// on the b component of ciphertexts [n][2][L][N]: b_j += enc_j(x0[n]).
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16) k_ntt_fwd(const uint64_t* in, uint64_t* out, const __grid_constant__ DevConsts c,
                                                             const uint64_t* __restrict__ x0) {
  constexpr int N = 1 << LOGN, T = N / 16;
  extern __shared__ uint64_t sm[];
  const size_t p = blockIdx.x;
  const int j = (int)(p % c.L);
  const uint64_t q = c.q[j], q2 = c.q2[j];
  const uint64_t* src = in + p * N;
  const bool share = x0 != nullptr && ((p / c.L) & 1);
  const uint64_t* xs = share ? x0 + (p / (2 * c.L)) * N : nullptr;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    uint64_t v = src[e];
    if (share) v += enc_lazy(__ldg(&xs[e]), j, c);  // < 4q: a valid lazy CT input
    sm[swz(e)] = v;
  }
  __syncthreads();
  ntt_fwd_smem<LOGN>(sm, c.tw_fwd + (size_t)j * N, q, q2);
  uint64_t* dst = out + p * N;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    dst[e] = csub(csub(sm[swz(e)], q2), q);
  }
}

// K3 (+A7 fused): inverse NTT of limb-polys in place; if r != NULL, on the b component of
// ciphertexts [n][2][L][N]: b_j += enc_j(r[n]) after the transform.
template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16) k_ntt_inv(uint64_t* polys, const __grid_constant__ DevConsts c,
                                                             const uint64_t* __restrict__ r) {
  constexpr int N = 1 << LOGN, T = N / 16;
  extern __shared__ uint64_t sm[];
  const size_t p = blockIdx.x;
  const int j = (int)(p % c.L);
  const uint64_t q = c.q[j], q2 = c.q2[j];
  uint64_t* buf = polys + p * N;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    sm[swz(e)] = buf[e];
  }
  __syncthreads();
  ntt_inv_smem<LOGN>(sm, c.tw_inv + (size_t)j * N, q, q2, c.ninv[j], c.ninv_p[j], c.wlast[j], c.wlast_p[j]);
  const bool mask = r != nullptr && ((p / c.L) & 1);
  const uint64_t* rs = mask ? r + (p / (2 * c.L)) * N : nullptr;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint32_t e = threadIdx.x + k * T;
    uint64_t v = sm[swz(e)];  // [0, 2q)
    if (mask) {
      v += enc_lazy(__ldg(&rs[e]), j, c);  // [0, 5q)
      v = csub(v, 2 * q2);
      v = csub(v, q2);
    }
    buf[e] = csub(v, q);
  }
}

// ------------------------------------------------------------------------------------------
// A4: NTT-domain multiply-accumulate ("performs all HE MAC operations in NTT"):
//   Y^[m,s,c,j,e] = sum_g X^[g,s,c,j,e] * W[m,g,j,e] mod q_j
// One thread owns 2 adjacent coefficients (128-bit loads) of limb j; its X^ values for the
// CTA's s-group are staged once in shared memory (thread-private columns, conflict-free) and
// reused for every m of the CTA's m-tile, so W streams from HBM exactly once and X^ is read
// from L2 once per m-tile. Products accumulate lazily in 128 bits, one reduction per output.
constexpr int MAC_THREADS = 128;

template <int SG>
__global__ void __launch_bounds__(MAC_THREADS) k_mac(const uint64_t* __restrict__ xhat,
                                                    const uint64_t* __restrict__ w, uint64_t* __restrict__ y,
                                                    const __grid_constant__ DevConsts c, PlanDev pl, int m_tile, int n_mtiles) {
  extern __shared__ ulonglong2 xs[];  // [G][2*SG][MAC_THREADS]
  const int N = 1 << c.log_n, L = c.L, G = pl.G, S = pl.S;
  const int j = blockIdx.y;
  const uint32_t e = (blockIdx.x * MAC_THREADS + threadIdx.x) * 2;
  const int mt = blockIdx.z % n_mtiles, sgi = blockIdx.z / n_mtiles;
  const int s0 = sgi * SG;
  const int ns = min(SG, S - s0);
  const uint64_t q = c.q[j];
  for (int g = 0; g < G; ++g)
    for (int sl = 0; sl < ns; ++sl)
      for (int cc = 0; cc < 2; ++cc)
        xs[(g * 2 * SG + sl * 2 + cc) * MAC_THREADS + threadIdx.x] = __ldg(reinterpret_cast<const ulonglong2*>(
            xhat + ((((size_t)g * S + s0 + sl) * 2 + cc) * L + j) * N + e));
  const int m_end = min((int)pl.M, (mt + 1) * m_tile);
  for (int m = mt * m_tile; m < m_end; ++m) {
    uint64_t lo[2 * SG][2], hi[2 * SG][2];
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a) lo[a][0] = lo[a][1] = hi[a][0] = hi[a][1] = 0;
    const uint64_t* wm = w + ((size_t)m * G * L + j) * N + e;
    for (int g = 0; g < G; ++g) {
      const ulonglong2 wv = __ldg(reinterpret_cast<const ulonglong2*>(wm + (size_t)g * L * N));
#pragma unroll
      for (int a = 0; a < 2 * SG; ++a) {
        if (a < 2 * ns) {
          const ulonglong2 xv = xs[(g * 2 * SG + a) * MAC_THREADS + threadIdx.x];
          mac128(lo[a][0], hi[a][0], xv.x, wv.x);
          mac128(lo[a][1], hi[a][1], xv.y, wv.y);
        }
      }
      if (g % 62 == 61) {  // keep the 128-bit sums below 2^128 (q < 2^61)
#pragma unroll
        for (int a = 0; a < 2 * SG; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            lo[a][b] = reduce128(lo[a][b], hi[a][b], q, c.r64[j], c.r64_p[j], c.one_p[j]);
            hi[a][b] = 0;
          }
      }
    }
#pragma unroll
    for (int a = 0; a < 2 * SG; ++a) {
      if (a < 2 * ns) {
        const int sl = a >> 1, cc = a & 1;
        ulonglong2 o;
        o.x = reduce128(lo[a][0], hi[a][0], q, c.r64[j], c.r64_p[j], c.one_p[j]);
        o.y = reduce128(lo[a][1], hi[a][1], q, c.r64[j], c.r64_p[j], c.one_p[j]);
        *reinterpret_cast<ulonglong2*>(y + ((((size_t)m * S + s0 + sl) * 2 + cc) * L + j) * N + e) = o;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// A3 packing: kernel [M][C][kh][kw] (< 2^t) -> mirrored coefficient-domain polys
// w[m][g][j][O - c*Hw*Ww - l*Ww - l'] = lift_j(K[m, g*Cw+c, l, l']) (reading R3: centred lift).
// The target must be zero-filled before.
__global__ void k_pack_weights(const uint64_t* __restrict__ kern, uint64_t* __restrict__ w, const __grid_constant__ DevConsts c,
                               PlanDev pl) {
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
    const uint64_t lifted = v >= t / 2 ? c.q[j] - (t - v) : v;  // t < q_j (checked at ctx creation)
    w[(((size_t)m * pl.G + g) * c.L + j) * N + coef] = lifted;
  }
}

// A6 / A7 standalone: ct [n][2][L][N], b_j += enc_j(v[n][N]).
__global__ void k_enc_add(uint64_t* __restrict__ ct, const uint64_t* __restrict__ v, const __grid_constant__ DevConsts c, size_t n) {
  const size_t N = 1ull << c.log_n;
  const size_t total = n * c.L * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t e = idx % N;
    const uint32_t j = (idx / N) % c.L;
    const size_t i = idx / (N * c.L);
    uint64_t* b = ct + ((i * 2 + 1) * c.L + j) * N + e;
    const uint64_t q = c.q[j];
    uint64_t s = *b + enc_lazy(v[i * N + e], j, c);  // [0, 4q)
    s = csub(s, 2 * q);
    *b = csub(s, q);
  }
}

// Designated server share y0[m][oy][ox] = (t - r[m*S+s][O + i*Ww + j]) mod t.
__global__ void k_extract_share(const uint64_t* __restrict__ r, uint64_t* __restrict__ y0, const __grid_constant__ DevConsts c, PlanDev pl) {
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

// SECN_VALIDATE: kind 0 = residues (limb-polys [P][N], limb p mod L, must be < q_j),
// kind 1 = plaintext-side values [n] (must be < 2^t_bits). Sets *flag on a violation.
__global__ void k_check_range(const uint64_t* __restrict__ v, size_t n_words, const __grid_constant__ DevConsts c, int kind,
                              uint32_t* flag) {
  const size_t N = 1ull << c.log_n;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n_words; idx += (size_t)gridDim.x * blockDim.x) {
    const uint64_t bound = kind == 0 ? c.q[(idx / N) % c.L] : (1ull << c.t_bits);
    if (v[idx] >= bound) *flag = 1;
  }
}

// ------------------------------------------------------------------------------------------
// launchers

template <int LOGN>
static cudaError_t ntt_fwd_t(const DevConsts& c, const uint64_t* in, uint64_t* out, size_t P, const uint64_t* x0,
                             cudaStream_t s) {
  constexpr int N = 1 << LOGN;
  const size_t smem = N * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ntt_fwd<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (size_t off = 0; off < P; off += 0x7fffffff) {
    const size_t cnt = P - off < 0x7fffffff ? P - off : 0x7fffffff;
    k_ntt_fwd<LOGN><<<(unsigned)cnt, N / 16, smem, s>>>(in + off * N, out + off * N, c, x0);
  }
  return cudaGetLastError();
}

cudaError_t launch_ntt_fwd(const DevConsts& c, const uint64_t* in, uint64_t* out, size_t P, const uint64_t* x0,
                           cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  switch (c.log_n) {
    case 12: return ntt_fwd_t<12>(c, in, out, P, x0, s);
    case 13: return ntt_fwd_t<13>(c, in, out, P, x0, s);
    case 14: return ntt_fwd_t<14>(c, in, out, P, x0, s);
  }
  return cudaErrorInvalidValue;
}

template <int LOGN>
static cudaError_t ntt_inv_t(const DevConsts& c, uint64_t* polys, size_t P, const uint64_t* r, cudaStream_t s) {
  constexpr int N = 1 << LOGN;
  const size_t smem = N * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ntt_inv<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  for (size_t off = 0; off < P; off += 0x7fffffff) {
    const size_t cnt = P - off < 0x7fffffff ? P - off : 0x7fffffff;
    k_ntt_inv<LOGN><<<(unsigned)cnt, N / 16, smem, s>>>(polys + off * N, c, r);
  }
  return cudaGetLastError();
}

cudaError_t launch_ntt_inv(const DevConsts& c, uint64_t* polys, size_t P, const uint64_t* r, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  switch (c.log_n) {
    case 12: return ntt_inv_t<12>(c, polys, P, r, s);
    case 13: return ntt_inv_t<13>(c, polys, P, r, s);
    case 14: return ntt_inv_t<14>(c, polys, P, r, s);
  }
  return cudaErrorInvalidValue;
}

template <int SG>
static cudaError_t mac_t(const DevConsts& c, const PlanDev& p, const uint64_t* xhat, const uint64_t* w, uint64_t* y,
                         cudaStream_t s) {
  const int N = 1 << c.log_n;
  const size_t smem = (size_t)p.G * 2 * SG * MAC_THREADS * sizeof(ulonglong2);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_mac<SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  const int m_tile = 16;
  const int n_mtiles = (p.M + m_tile - 1) / m_tile;
  const int n_sg = (p.S + SG - 1) / SG;
  dim3 grid(N / (2 * MAC_THREADS), c.L, n_mtiles * n_sg);
  k_mac<SG><<<grid, MAC_THREADS, smem, s>>>(xhat, w, y, c, p, m_tile, n_mtiles);
  return cudaGetLastError();
}

cudaError_t launch_mac(const DevConsts& c, const PlanDev& p, const uint64_t* xhat, const uint64_t* w, uint64_t* y,
                       cudaStream_t s) {
  if (p.M == 0 || p.S == 0) return cudaSuccess;
  // s-group size: as many of the S blocks as fit 200 KiB of shared memory (at most 4).
  const size_t per_s = (size_t)p.G * 2 * MAC_THREADS * sizeof(ulonglong2);
  int sg = 4;
  while (sg > 1 && per_s * sg > 200 * 1024) --sg;
  if (per_s > 200 * 1024) return cudaErrorInvalidValue;  // G too large for one CTA (G > 50)
  if (sg > (int)p.S) sg = p.S;
  switch (sg) {
    case 1: return mac_t<1>(c, p, xhat, w, y, s);
    case 2: return mac_t<2>(c, p, xhat, w, y, s);
    case 3: return mac_t<3>(c, p, xhat, w, y, s);
    default: return mac_t<4>(c, p, xhat, w, y, s);
  }
}

cudaError_t launch_pack_weights(const DevConsts& c, const PlanDev& p, const uint64_t* kernel, uint64_t* w,
                                cudaStream_t s) {
  const size_t N = 1ull << c.log_n;
  cudaError_t e = cudaMemsetAsync(w, 0, (size_t)p.M * p.G * c.L * N * sizeof(uint64_t), s);
  if (e != cudaSuccess) return e;
  const size_t total = (size_t)p.M * p.C * p.kh * p.kw;
  if (total) k_pack_weights<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(kernel, w, c, p);
  return cudaGetLastError();
}

cudaError_t launch_enc_add(const DevConsts& c, uint64_t* ct, const uint64_t* v, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const size_t total = n * c.L * (1ull << c.log_n);
  const size_t blocks = (total + 255) / 256;
  k_enc_add<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, s>>>(ct, v, c, n);
  return cudaGetLastError();
}

cudaError_t launch_extract_share(const DevConsts& c, const PlanDev& p, const uint64_t* r, uint64_t* y0,
                                 cudaStream_t s) {
  const size_t total = (size_t)p.M * p.OH * p.OW;
  if (total) k_extract_share<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(r, y0, c, p);
  return cudaGetLastError();
}

cudaError_t launch_check_range(const DevConsts& c, const uint64_t* v, size_t n_words, int kind, uint32_t* flag,
                               cudaStream_t s) {
  if (n_words == 0) return cudaSuccess;
  const size_t blocks = (n_words + 255) / 256;
  k_check_range<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(v, n_words, c, kind, flag);
  return cudaGetLastError();
}

}  // namespace secn
