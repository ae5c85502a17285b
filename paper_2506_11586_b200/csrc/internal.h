// Internal declarations shared by api.cpp (host) and kernels.cu (device) of libsecn.
#pragma once
#include <cstddef>
#include <cstdint>
#include <mutex>

#include <cuda_runtime.h>

#include "../../include/secn.h"

namespace secn {

// Per-context constants passed by value to every kernel (kernel-parameter space).
// word_bits = 64: residues are uint64 (q < 2^61), twiddles in tw_fwd/tw_inv (Shoup w' over 2^64).
// word_bits = 32: residues are uint32 (q < 2^30), twiddles in tw32_fwd/tw32_inv (w' over 2^32).
// The 64-bit companions of delta / one_p are kept for both (encoding and reductions use 64-bit
// arithmetic in either case).
// Tuning knobs and device facts, read once at context creation (the SECN_* environment
// variables are developer knobs for tools/; every default is the measured best).
struct Tune {
  int32_t no_pdl;       // SECN_NO_PDL=1: plain stream order instead of programmatic dependent launch
  int32_t ntt_np2_min;  // SECN_NTT_NP2_MIN: limb-polys from which N = 4096 32-bit NTTs pair two polys per CTA
  int32_t ntt_tma;      // SECN_NTT_TMA: plain calls on the TMA-staged engine -- 0 never, 1 measured rule, 2 always
  int32_t ntt_tma_min;  // SECN_NTT_TMA_MIN: limb-polys from which the plain calls use the TMA-staged engine
  int32_t tail1;        // SECN_TAIL1=1: one-component INTT tail at N = 4096
  int32_t mac_kb;       // SECN_MAC_KB: k_mac shared-memory budget per CTA (KiB)
  int32_t mac_xamort;   // SECN_MAC_XAMORT=0: no X^-tile amortisation rule
  int32_t mac_nmr;      // SECN_MAC_NMR: forced m-range count
  int32_t mac_nohint;   // SECN_MAC_NOHINT=1: no L2 hint on the weight stream
  int32_t mac_pre;      // SECN_MAC_PRE: weight stages issued before the dependency wait (chained calls)
  int32_t mac_sg;       // SECN_MAC_SG / SECN_MAC_MT: forced k_mac register block
  int32_t mac_mt;
  int32_t mac_ws;       // SECN_MAC_WS: the warp-specialised k_mac_ws (32-bit limbs): 0 never, 1 rule, 2 always
  int32_t fused;        // SECN_FUSED=2: the fused small-layer kernel for every layer it supports (default 0: off)
  int32_t fused_sg;     // SECN_FUSED_SG / SECN_FUSED_MT: its register block (s-group, m-block)
  int32_t fused_mt;
  int32_t fused_kb;     // SECN_FUSED_KB: its shared-memory budget per CTA (KiB)
  int32_t validate;     // SECN_VALIDATE=1: range-check input values (synchronous)
  int32_t num_sms;      // multiprocessor count of the context's device
};

struct DevConsts {
  uint64_t q[SECN_MAX_LIMBS];
  uint64_t ninv[SECN_MAX_LIMBS], ninv_p[SECN_MAX_LIMBS];    // N^-1 (Shoup, word-sized companion)
  uint64_t wlast[SECN_MAX_LIMBS], wlast_p[SECN_MAX_LIMBS];  // psi^-brv(1) N^-1 (Shoup, word-sized)
  uint64_t delta[SECN_MAX_LIMBS], delta_p[SECN_MAX_LIMBS];  // floor(Q/t) mod q (Shoup over 2^64)
  uint64_t r64[SECN_MAX_LIMBS], r64_p[SECN_MAX_LIMBS];      // 2^64 mod q (Shoup over 2^64)
  uint64_t one_p[SECN_MAX_LIMBS];                           // floor(2^64 / q)
  uint64_t tinv[SECN_MAX_LIMBS], tinv_p[SECN_MAX_LIMBS];    // t^-1 mod q (Shoup, word-sized companion)
  uint64_t tinv_hi[SECN_MAX_LIMBS], tinv_hi_p[SECN_MAX_LIMBS];  // 2^32 t^-1 mod q (32-bit limbs)
  uint64_t r32[SECN_MAX_LIMBS], r32_p[SECN_MAX_LIMBS];      // 2^32 mod q (32-bit Shoup; 32-bit limbs)
  uint64_t qmt;                                             // Q mod t
  uint32_t t_bits, log_n, L, word_bits;
  const ulonglong2* tw_fwd;  // [L][N] (psi^brv(i), w')      word_bits = 64
  const ulonglong2* tw_inv;  // [L][N] (psi^-brv(i), w')
  const uint2* tw32_fwd;     // [L][N]                        word_bits = 32
  const uint2* tw32_inv;
  // N = 2^15 only: per-half tables [L][2][N/2] for the two 2^14-point halves of the cluster NTT:
  // th[k] = t[k + hp2(k) (1 + h)], hp2(k) = the largest power of two <= k (k >= 1)
  const ulonglong2* tw_fwd_h;
  const ulonglong2* tw_inv_h;
  const uint2* tw32_fwd_h;
  const uint2* tw32_inv_h;
  uint64_t one_wp[SECN_MAX_LIMBS];  // word-sized Shoup companion of 1
  // inverse NTT after the NTT-domain MAC (k_mac's outputs): when mac_redc, k_mac reduces the MAC
  // sums by Montgomery REDC (x 2^-32), so these are N^-1 2^32 and psi^-brv(1) N^-1 2^32
  // (otherwise equal to ninv / wlast); qneg_inv32 = -q^-1 mod 2^32
  uint64_t ninv_mac[SECN_MAX_LIMBS], ninv_mac_p[SECN_MAX_LIMBS];
  uint64_t wlast_mac[SECN_MAX_LIMBS], wlast_mac_p[SECN_MAX_LIMBS];
  uint64_t qneg_inv32[SECN_MAX_LIMBS];
  uint32_t mac_redc;  // 1: 32-bit limbs with every q < 2^27 (G q < 2^32 for G <= 32): k_mac uses REDC
  Tune tune;          // host-side launch choices (never read by a kernel)
};

struct PlanDev;
// the index m*S + s of the i-th output ciphertext of a call with an s-slice (i = m * sn + s - s0)
__host__ __device__ inline uint32_t slice_ct(const PlanDev& p, uint32_t i);

struct PlanDev {  // the subset of secn_conv_plan (kind 0) / secn_fc_plan (kind 1) the kernels use
  uint32_t M, G, S, Cw, Hw, Ww, kh, kw, C, O, OH, OW, nbh, nbw, sh;
  uint32_t kh0, kw0, ps;  // the caller's kernel extent and the polyphase factor (reading R7b; kh, kw
                          // above are the window's extent ceil(kh0/ps) x ceil(kw0/ps))
  uint32_t kind;         // 0: convolution, 1: fully connected (S = 1)
  uint32_t s0, sn;       // output spatial-block slice [s0, s0 + sn) of S (sn = S: all)
  uint32_t nib, nob, no; // fc: inputs per ct, output rows per ct, n_o (C holds n_i)
};

// Reading R17: the device-drawn mask (secn_mask_gen_t): Philox4x32-10 keyed by seed, counter
// (coefficient pair, ct0 + output ct, stream, 0).
struct MaskGen {
  uint64_t seed;
  uint32_t stream, ct0;
};

__host__ __device__ inline uint32_t slice_ct(const PlanDev& p, uint32_t i) {
  return p.sn == p.S ? i : (i / p.sn) * p.S + p.s0 + i % p.sn;
}

// Modulus switch Q -> Q' = q_0 .. q_{Lk-1} (reading R16): P = the product of the dropped primes
// q_Lk .. q_{L-1}; for a dropped limb j: pq[j] = P / q_j and inv[j] = (P / q_j)^-1 mod q_j; for a
// kept limb i: pinv[i] = P^-1 mod q_i (companions word-sized). Built per call on the host.
struct MsConsts {
  uint32_t Lk;
  uint64_t P;
  uint64_t pq[SECN_MAX_LIMBS], inv[SECN_MAX_LIMBS], inv_p[SECN_MAX_LIMBS];
  uint64_t pinv[SECN_MAX_LIMBS], pinv_p[SECN_MAX_LIMBS];
};

// ---- launchers (kernels.cu); all return cudaGetLastError() after the launch(es) ----
// Reads the tuning knobs (environment) and the device's SM count into *t.
void read_tune(int device, Tune* t);
// Opts every shared-memory-hungry kernel of this word size into the full 227 KiB of dynamic shared
// memory on the CURRENT device (function attributes are per device): called by secn_ctx_create.
cudaError_t init_device(uint32_t word_bits);
//
// Pre-wait reads. Under programmatic dependent launch a kernel starts while its predecessor in the
// stream finishes; it may read an input before griddepcontrol.wait only if that predecessor is
// known not to produce it. `chained` = true says the predecessor is the preceding launch of the
// same library call (which waits for its own predecessor before triggering and never writes the
// weights or the mask), so k_mac may pre-issue weight loads and the tails may load the mask early;
// a stage call on its own passes false.
// Residue buffers are void* of the context's word size.
cudaError_t launch_ntt_fwd(const DevConsts& c, const void* in, void* out, size_t n_limb_polys, const uint64_t* x0,
                           cudaStream_t s);
cudaError_t launch_ntt_inv(const DevConsts& c, void* polys, size_t n_limb_polys, cudaStream_t s);
// levels 8.. of the inverse NTT (+N^-1, +mask) after launch_mac applied levels 0..7; if
// y0 != NULL also the server share (A8) for plan pl
// em != NULL: the mask arrives encoded (k_mask_encode's em [rows][L][N]); r and y0 are then unused
cudaError_t launch_ntt_inv_tail(const DevConsts& c, void* polys, size_t n_limb_polys, const uint64_t* r, uint64_t* y0,
                                const PlanDev& pl, cudaStream_t s, bool chained, const void* em = nullptr);
// The whole layer after the forward NTT in one kernel (32-bit limbs, N = 4096): A4 MAC, the full
// inverse NTT, A7 mask, A8 share. fused_applies says whether the layer takes this path.
bool fused_applies(const DevConsts& c, const PlanDev& p);
cudaError_t launch_layer_fused(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y,
                               const uint64_t* r, uint64_t* y0, cudaStream_t s, bool chained, const void* em);
// NTT-domain MAC (A4) followed by inverse-NTT levels 0..7 of its outputs (lazy GS domain)
cudaError_t launch_mac(const DevConsts& c, const PlanDev& p, const void* xhat, const void* w, void* y, cudaStream_t s,
                       bool chained);
cudaError_t launch_pack_weights(const DevConsts& c, const PlanDev& p, const uint64_t* kernel, void* w, cudaStream_t s);
// f2: levels 8.. of the inverse NTT + mask + modulus switch to ms.Lk limbs + extraction, N = 4096
// only: polys [n_ct][2][L][N] (after launch_mac) -> a_out [n_ct][Lk][N], b_out [values][Lk] at the
// designated coefficients of plan pl (conv or fc), and y0 (if not NULL) the server share.
cudaError_t launch_ntt_inv_tail_lwe(const DevConsts& c, const MsConsts& ms, const void* polys, size_t n_ct,
                                    const uint64_t* r, void* a_out, void* b_out, uint64_t* y0, const PlanDev& pl,
                                    cudaStream_t s, bool chained, const void* em = nullptr);
// fc weights W [n_o][n_i] -> mirrored polys [M][G][L][N] (coefficient domain, zero-filled first)
cudaError_t launch_pack_fc_weights(const DevConsts& c, const PlanDev& p, const uint64_t* W, void* w, cudaStream_t s);
// r [n_ct][N] from the generator (reading R17); launched with PDL, safe to chain (see k_mask_draw)
cudaError_t launch_mask_draw(const DevConsts& c, const MaskGen& g, size_t n_ct, uint64_t* r, cudaStream_t s);
// em [rows][L][N] (word size) = enc_j(r) of the call's n_act output ciphertexts (rows slice_ct),
// r from `r` (device) or, if r == NULL, drawn by g; y0 (may be NULL) = -r mod t at the designated
// outputs. chained: launched right after the forward NTT of the same call (waits for it only at the
// end, so that the MAC's dependency wait covers both); else a standalone call (waits first).
cudaError_t launch_mask_encode(const DevConsts& c, const PlanDev& p, size_t n_act, const uint64_t* r, const MaskGen& g,
                               void* em, uint64_t* y0, cudaStream_t s, bool chained);
cudaError_t launch_enc_add(const DevConsts& c, void* ct, const uint64_t* v, size_t n, cudaStream_t s);
cudaError_t launch_extract_share(const DevConsts& c, const PlanDev& p, const uint64_t* r, uint64_t* y0,
                                 cudaStream_t s);
// kind 0: residues (n_words of the context's word size, limb = (idx / N) mod L, < q_j);
// kind 1: uint64 plaintext-side values (< 2^t_bits).
cudaError_t launch_check_range(const DevConsts& c, const void* v, size_t n_words, int kind, uint32_t* flag,
                               cudaStream_t s);

}  // namespace secn

struct secn_ctx {
  int device;
  uint32_t log_n, n, L, t_bits, word_bits;
  uint64_t primes[SECN_MAX_LIMBS], psi[SECN_MAX_LIMBS];
  secn::DevConsts dc;
  void* d_tables;
  uint32_t* d_flag;        // SECN_VALIDATE scratch
  std::mutex* flag_mutex;  // serialises the validated calls that share d_flag
};
