// Modular arithmetic policies for sm_100a (device side of libsecn).
//
// Arith64: residues in uint64, every modulus q < 2^61. Multiplication by a fixed operand w
// uses Shoup's precomputed companion w' = floor(w 2^64 / q) with a TRUNCATED quotient: the
// 64x64 high product omits the low x low partial product and the carries of the cross terms,
// so the quotient estimate is short by at most 2 and the result lies in [0, 4q) (instead of
// [0, 2q)) -- one 32x32 wide multiply and two carry chains cheaper on the integer pipes.
// Lazy domains (Harvey): Cooley-Tukey values live in [0, 8q), Gentleman-Sande values in
// [0, 4q); 8q < 2^64 because q < 2^61.
#pragma once
#include <cstdint>

namespace secn {

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }

// floor(a * b / 2^64) exactly
__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// floor(a * b / 2^64) - e, e in {0, 1, 2}: x1 p1 + hi(x1 p0) + hi(x0 p1)
__device__ __forceinline__ uint64_t mulhi_trunc(uint64_t x, uint64_t p) {
  const uint32_t x0 = lo32(x), x1 = hi32(x), p0 = lo32(p), p1 = hi32(p);
  const uint64_t s = (uint64_t)__umulhi(x1, p0) + __umulhi(x0, p1);
  return (uint64_t)x1 * p1 + s;
}

// Exact Shoup: x w mod q in [0, 2q) for any x < 2^64.
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  return x * w - mulhi(x, wp) * q;
}

// Truncated Shoup: x w mod q in [0, 4q) for any x < 2^64.
__device__ __forceinline__ uint64_t shoup4(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  return x * w - mulhi_trunc(x, wp) * q;
}

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

struct Arith64 {
  using W = uint64_t;
  using Tw = ulonglong2;  // (w, w')
  // lazy-domain bound used by csub in both butterflies: CT values in [0, 2*bound),
  // GS values in [0, bound)
  __device__ static __forceinline__ W bound(W q) { return 4 * q; }
  // Cooley-Tukey butterfly on [0, 8q): X, Y -> X + wY, X - wY.  q4 = 4q.
  __device__ static __forceinline__ void ct(W& X, W& Y, const Tw t, W q, W q4) {
    const W x = csub(X, q4);                 // [0, 4q)
    const W y = shoup4(Y, t.x, t.y, q);      // [0, 4q)
    X = x + y;                               // [0, 8q)
    Y = x - y + q4;                          // (0, 8q)
  }
  // Gentleman-Sande butterfly on [0, 4q): U, V -> U + V, (U - V) w.
  __device__ static __forceinline__ void gs(W& U, W& V, const Tw t, W q, W q4) {
    const W u = U, v = V;
    U = csub(u + v, q4);                     // [0, 4q)
    V = shoup4(u - v + q4, t.x, t.y, q);     // [0, 4q)
  }
  // x w mod q in [0, 4q) for any x < 2^64
  __device__ static __forceinline__ W mul4(W x, const Tw t, W q) { return shoup4(x, t.x, t.y, q); }
  // CT domain [0, 8q) -> [0, q)
  __device__ static __forceinline__ W canon_ct(W x, W q) { return csub(csub(csub(x, 4 * q), 2 * q), q); }
  // GS domain [0, 4q) -> [0, q)
  __device__ static __forceinline__ W canon_gs(W x, W q) { return csub(csub(x, 2 * q), q); }
};

// Arith32: residues in uint32, every modulus q < 2^30 (32-bit RNS limbs).
// Exact Shoup with w' = floor(w 2^32 / q): one IMAD.HI + two IMADs. Harvey domains: CT values in
// [0, 4q), GS values in [0, 2q). csub(x, m) = min(x, x - m) (unsigned wrap) is one IADD + one
// VIMNMX.
__device__ __forceinline__ uint32_t csub32(uint32_t x, uint32_t m) { return min(x, x - m); }

struct Arith32 {
  using W = uint32_t;
  using Tw = uint2;  // (w, w')
  __device__ static __forceinline__ W bound(W q) { return 2 * q; }
  __device__ static __forceinline__ W shoup32(W x, W w, W wp, W q) { return x * w - __umulhi(x, wp) * q; }
  // CT butterfly on [0, 4q).  qb = 2q.
  __device__ static __forceinline__ void ct(W& X, W& Y, const Tw t, W q, W qb) {
    const W x = csub32(X, qb);             // [0, 2q)
    const W y = shoup32(Y, t.x, t.y, q);   // [0, 2q)
    X = x + y;                             // [0, 4q)
    Y = x - y + qb;                        // (0, 4q)
  }
  // GS butterfly on [0, 2q).
  __device__ static __forceinline__ void gs(W& U, W& V, const Tw t, W q, W qb) {
    const W u = U, v = V;
    U = csub32(u + v, qb);                 // [0, 2q)
    V = shoup32(u - v + qb, t.x, t.y, q);  // [0, 2q)
  }
  __device__ static __forceinline__ W mul4(W x, const Tw t, W q) { return shoup32(x, t.x, t.y, q); }
  __device__ static __forceinline__ W canon_ct(W x, W q) { return csub32(csub32(x, 2 * q), q); }
  __device__ static __forceinline__ W canon_gs(W x, W q) { return csub32(x, q); }
};

// 128-bit accumulator (lo, hi) += a * b.
__device__ __forceinline__ void mac128(uint64_t& lo, uint64_t& hi, uint64_t a, uint64_t b) {
  const uint64_t pl = a * b, ph = mulhi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(pl), "l"(ph));
}

// (hi * 2^64 + lo) mod q, canonical. r64 = 2^64 mod q with Shoup companion r64p;
// onep = floor(2^64 / q) (the Shoup companion of 1).
__device__ __forceinline__ uint64_t reduce128(uint64_t lo, uint64_t hi, uint64_t q, uint64_t r64, uint64_t r64p,
                                              uint64_t onep) {
  const uint64_t a = shoup(hi, r64, r64p, q);   // [0, 2q)
  const uint64_t b = lo - mulhi(lo, onep) * q;  // [0, 2q)
  uint64_t s = a + b;                           // [0, 4q)
  s = csub(s, 2 * q);
  return csub(s, q);
}

}  // namespace secn
