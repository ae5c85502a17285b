/*
 * SecONNds HE-convolution ORACLE -- plain, slow, obviously-correct CPU reference.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code, header,
 * table or constant generator with the CUDA path (paper_2506_11586_b200/), and the CUDA
 * path never loads it.
 *
 * Every function computes a plain definition with unsigned __int128 arithmetic and one
 * `%` reduction per product; there is no blocking, lazy reduction, Shoup/Barrett
 * precomputation or NTT anywhere in this file.
 *
 *   orc_negacyclic_mul   c = a * b in Z_q[X]/(X^N+1)           PAPER.md:60 (§2.1 ring),
 *                        schoolbook over all i, j               PAPER.md:661-667 (App. C; the
 *                                                               printed sum is the acyclic half,
 *                                                               DESIGN.md reading R12)
 *   orc_ntt_direct       A[k] = sum_i a_i psi^((2 brv(k)+1) i)  PAPER.md:668-679 (App. C.1),
 *                                                               bit-reversed order: reading R4
 *   orc_intt_direct      a_i = N^-1 sum_k A[k] psi^-((2brv(k)+1) i)   (inverse of the above)
 *   orc_enc              enc_j(v) = round(Q v / t) mod q_j      PAPER.md:654 (App. C, delta*m),
 *                                                               reading R2 (round, not floor)
 *   orc_he_conv_server   out[m,s] = sum_g in'[g,s] (*) lift(w[m,g]) (+ enc(r) on b)
 *                                                               PAPER.md:380 (§6.2), :431 (§7)
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o liboracle.so oracle.c
 */
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + b) % q); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a + q - b) % q); }

uint64_t orc_powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = mulmod(r, b, q);
    b = mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}

static uint32_t brv(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

/* c[k] = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j  (mod q)  -- the negacyclic product. */
void orc_negacyclic_mul(const uint64_t* a, const uint64_t* b, uint64_t* c, uint32_t n, uint64_t q) {
  for (uint32_t k = 0; k < n; ++k) c[k] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (a[i] == 0) continue;
    for (uint32_t j = 0; j < n; ++j) {
      uint64_t p = mulmod(a[i], b[j], q);
      uint32_t k = i + j;
      if (k < n) c[k] = addmod(c[k], p, q);
      else c[k - n] = submod(c[k - n], p, q); /* X^N = -1 */
    }
  }
}

/* Forward negacyclic NTT by direct evaluation at the N odd powers of psi, output entry k
 * holding a(psi^(2 brv(k) + 1)).  O(N^2). */
void orc_ntt_direct(const uint64_t* a, uint64_t* out, uint32_t logn, uint64_t q, uint64_t psi) {
  uint32_t n = 1u << logn;
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t zeta = orc_powmod(psi, 2 * (uint64_t)brv(k, logn) + 1, q);
    uint64_t acc = 0, p = 1;
    for (uint32_t i = 0; i < n; ++i) {
      acc = addmod(acc, mulmod(a[i], p, q), q);
      p = mulmod(p, zeta, q);
    }
    out[k] = acc;
  }
}

/* Same definition, only at the requested output indices ks[0..nk). */
void orc_ntt_direct_sampled(const uint64_t* a, const uint32_t* ks, uint64_t* out, size_t nk, uint32_t logn,
                            uint64_t q, uint64_t psi) {
  uint32_t n = 1u << logn;
  for (size_t t = 0; t < nk; ++t) {
    uint64_t zeta = orc_powmod(psi, 2 * (uint64_t)brv(ks[t], logn) + 1, q);
    uint64_t acc = 0, p = 1;
    for (uint32_t i = 0; i < n; ++i) {
      acc = addmod(acc, mulmod(a[i], p, q), q);
      p = mulmod(p, zeta, q);
    }
    out[t] = acc;
  }
}

/* Inverse: a_i = N^-1 * sum_k A[k] * zeta_k^-i, zeta_k = psi^(2 brv(k)+1).  O(N^2). */
void orc_intt_direct(const uint64_t* A, uint64_t* out, uint32_t logn, uint64_t q, uint64_t psi) {
  uint32_t n = 1u << logn;
  uint64_t n_inv = orc_powmod(n, q - 2, q);   /* q prime: Fermat inverse */
  uint64_t psi_inv = orc_powmod(psi, q - 2, q);
  for (uint32_t i = 0; i < n; ++i) out[i] = 0;
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t zinv = orc_powmod(psi_inv, 2 * (uint64_t)brv(k, logn) + 1, q);
    uint64_t p = 1;
    for (uint32_t i = 0; i < n; ++i) {
      out[i] = addmod(out[i], mulmod(A[k], p, q), q);
      p = mulmod(p, zinv, q);
    }
  }
  for (uint32_t i = 0; i < n; ++i) out[i] = mulmod(out[i], n_inv, q);
}

/* enc_j(v) = round(Q v / t) mod q_j with round-half-up (reading R2/R5), t = 2^t_bits.
 * Q v / t = floor(Q/t) v + (Q mod t) v / t, so
 * round(Q v / t) = floor(Q/t) v + floor(((Q mod t) v + t/2) / t).
 * delta_mod_q = floor(Q/t) mod q_j and q_mod_t = Q mod t are passed in (computed with
 * Python big integers in oracle/params.py). */
static uint64_t enc_one(uint64_t v, uint64_t q, uint64_t delta_mod_q, uint64_t q_mod_t, uint32_t t_bits) {
  u128 frac = ((u128)q_mod_t * v + ((u128)1 << (t_bits - 1))) >> t_bits;
  return addmod(mulmod(delta_mod_q, v % q, q), (uint64_t)(frac % q), q);
}

void orc_enc(const uint64_t* v, uint64_t* out, size_t n, uint64_t q, uint64_t delta_mod_q, uint64_t q_mod_t,
             uint32_t t_bits) {
  for (size_t i = 0; i < n; ++i) out[i] = enc_one(v[i], q, delta_mod_q, q_mod_t, t_bits);
}

/* lift_j(w): the centred representative of w mod t, in [-t/2, t/2), reduced mod q_j
 * (reading R3). */
static uint64_t lift(uint64_t w, uint64_t q, uint32_t t_bits) {
  uint64_t t = (uint64_t)1 << t_bits;
  if (w >= t / 2) return submod(0, (t - w) % q, q);
  return w % q;
}

/*
 * Server side of one HE convolution layer in the coefficient domain (no NTT):
 *
 *   in'[g,s].b_j = in[g,s].b_j + enc_j(x0[g,s])            if x0 != NULL
 *   out[m,s].c_j = sum_{g<G} in'[g,s].c_j (*) lift_j(w[m,g])  in Z_qj[X]/(X^N+1)
 *   out[m,s].b_j += enc_j(r[m,s])                          if r != NULL
 *
 * ct_in  : [G*S][2][L][N]  (index g*S+s; component 0 = a, 1 = b)
 * x0     : [G*S][N] or NULL, values < 2^t_bits
 * kernel polys (m,g) in sparse form: nonzero coefficient indices kidx[koff[mg] .. koff[mg+1])
 *          with raw values kval (< 2^t_bits), mg = m*G+g. Skipping zero coefficients of the
 *          schoolbook sum does not change it.
 * r      : [M*S][N] or NULL
 * out    : [M*S][2][L][N]
 * Only outputs (m,s) with sel == NULL or sel[m*S+s] != 0 are computed (others untouched):
 * the bench samples a bounded subset of outputs.
 */
void orc_he_conv_server(uint32_t logn, uint32_t L, const uint64_t* primes, uint32_t t_bits,
                        const uint64_t* delta_mod_q, uint64_t q_mod_t, uint32_t G, uint32_t S, uint32_t M,
                        const uint64_t* ct_in, const uint64_t* x0, const uint64_t* koff, const uint32_t* kidx,
                        const uint64_t* kval, const uint64_t* r, const uint8_t* sel, uint64_t* out) {
  const size_t n = (size_t)1 << logn;
  const long long n_out = (long long)M * S;
#pragma omp parallel
  {
    uint64_t* acc = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* inb = (uint64_t*)malloc(n * sizeof(uint64_t));
#pragma omp for schedule(dynamic, 1)
    for (long long ms = 0; ms < n_out; ++ms) {
      if (sel && !sel[ms]) continue;
      const uint32_t m = (uint32_t)(ms / S), s = (uint32_t)(ms % S);
      for (uint32_t c = 0; c < 2; ++c) {
        for (uint32_t j = 0; j < L; ++j) {
          const uint64_t q = primes[j];
          for (size_t i = 0; i < n; ++i) acc[i] = 0;
          for (uint32_t g = 0; g < G; ++g) {
            const uint64_t* src = ct_in + (((size_t)(g * S + s) * 2 + c) * L + j) * n;
            /* server-share add on the b component */
            for (size_t i = 0; i < n; ++i) {
              inb[i] = src[i];
              if (c == 1 && x0) inb[i] = addmod(inb[i], enc_one(x0[(size_t)(g * S + s) * n + i], q, delta_mod_q[j], q_mod_t, t_bits), q);
            }
            const size_t mg = (size_t)m * G + g;
            for (uint64_t z = koff[mg]; z < koff[mg + 1]; ++z) {
              const uint32_t d = kidx[z];
              const uint64_t w = lift(kval[z], q, t_bits);
              for (size_t i = 0; i < n; ++i) {
                const uint64_t p = mulmod(inb[i], w, q);
                const size_t k = i + d;
                if (k < n) acc[k] = addmod(acc[k], p, q);
                else acc[k - n] = submod(acc[k - n], p, q); /* X^N = -1 */
              }
            }
          }
          if (c == 1 && r) {
            for (size_t i = 0; i < n; ++i)
              acc[i] = addmod(acc[i], enc_one(r[(size_t)ms * n + i], q, delta_mod_q[j], q_mod_t, t_bits), q);
          }
          memcpy(out + (((size_t)ms * 2 + c) * L + j) * n, acc, n * sizeof(uint64_t));
        }
      }
    }
    free(acc);
    free(inb);
  }
}

int orc_num_threads(void) {
  int t = 1;
#pragma omp parallel
  {
#pragma omp single
    {
#ifdef _OPENMP
      t = omp_get_num_threads();
#endif
    }
  }
  return t;
}
