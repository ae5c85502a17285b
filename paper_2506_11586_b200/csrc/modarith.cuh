// 64-bit modular arithmetic for sm_100a (device side of libsecn).
//
// All moduli satisfy q < 2^61 (checked at context creation), so the lazy ranges used below
// ([0, 4q) for Cooley-Tukey, [0, 2q) for Gentleman-Sande, 128-bit sums of up to 63 products)
// never overflow a 64-bit word.
#pragma once
#include <cstdint>

namespace secn {

// floor(a * b / 2^64)
__device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// Shoup multiplication by a fixed operand w < q with companion wp = floor(w * 2^64 / q):
// returns x * w mod q up to one extra q, i.e. a value in [0, 2q), for ANY x < 2^64.
__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  return x * w - mulhi(x, wp) * q;
}

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) { return x >= m ? x - m : x; }

// Harvey lazy Cooley-Tukey butterfly: X, Y in [0, 4q) -> X + wY, X - wY in [0, 4q).
__device__ __forceinline__ void ct_bfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t wp, uint64_t q,
                                        uint64_t q2) {
  const uint64_t x = csub(X, q2);
  const uint64_t t = shoup(Y, w, wp, q);
  X = x + t;
  Y = x - t + q2;
}

// Harvey lazy Gentleman-Sande butterfly: U, V in [0, 2q) -> U + V, (U - V) w in [0, 2q).
__device__ __forceinline__ void gs_bfly(uint64_t& U, uint64_t& V, uint64_t w, uint64_t wp, uint64_t q,
                                        uint64_t q2) {
  const uint64_t u = U, v = V;
  U = csub(u + v, q2);
  V = shoup(u - v + q2, w, wp, q);
}

// 128-bit accumulator (lo, hi) += a * b.
__device__ __forceinline__ void mac128(uint64_t& lo, uint64_t& hi, uint64_t a, uint64_t b) {
  const uint64_t pl = a * b, ph = mulhi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(pl), "l"(ph));
}

// (hi * 2^64 + lo) mod q, canonical. r64 = 2^64 mod q with Shoup companion r64p;
// onep = floor(2^64 / q) (the Shoup companion of 1).
__device__ __forceinline__ uint64_t reduce128(uint64_t lo, uint64_t hi, uint64_t q, uint64_t r64, uint64_t r64p,
                                              uint64_t onep) {
  const uint64_t a = shoup(hi, r64, r64p, q);  // [0, 2q)
  const uint64_t b = lo - mulhi(lo, onep) * q;  // [0, 2q)
  uint64_t s = a + b;                           // [0, 4q)
  s = csub(s, 2 * q);
  return csub(s, q);
}

}  // namespace secn
