/*
 * secn.h -- C ABI of libsecn, the B200 (sm_100a) server-side homomorphic linear layer of
 * SecONNds (arXiv 2506.11586): Cheetah-style coefficient-encoded convolution on RLWE/BFV
 * ciphertexts with NTT-preprocessed weights.
 *
 * Citations are PAPER.md line numbers (PAPER.md = the paper's LaTeX source) with the section;
 * "reading Rk" refers to DESIGN.md's list of readings where the paper is silent.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Ring R_Q = Z_Q[X]/(X^N+1) (§2.1), Q = q_0 ... q_{L-1} in RNS. A limb-poly is
 *    N uint64 residues mod one q_j; a poly is L limb-polys [L][N]; a ciphertext is (a, b) =
 *    [2][L][N] (App. C; index 0 = a, 1 = b). All arrays are row-major with
 *    the last index fastest and live in DEVICE memory of the context's device unless stated.
 *  - Every residue at the boundary is canonical, in [0, q_j). Plaintext-side values (server
 *    shares x0, masks r, kernel weights) are integers in [0, 2^t_bits).
 *  - NTT domain: entry k of a limb-poly holds a(psi_j^(2 brv(k) + 1)) with psi_j the smallest
 *    primitive 2N-th root mod q_j (bit-reversed order, reading R4; App. C.1).
 *  - Encoding (reading R2): enc_j(v) = round(Q v / t) mod q_j, round half up, t = 2^t_bits.
 *  - Ownership: the caller allocates and owns every I/O and workspace buffer and the stream.
 *    The library owns only the context's device tables (freed by secn_ctx_destroy).
 *  - Asynchrony: compute calls only enqueue work on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and return; device faults surface at the caller's next
 *    synchronisation. No call synchronises the device or allocates memory except
 *    secn_ctx_create / secn_ctx_destroy.
 *  - Errors: every call returns a secn_status; none throws or aborts. secn_last_error()
 *    returns a thread-local message for the last non-OK status of the calling thread.
 *  - Thread safety: a context is immutable after creation; concurrent calls on different
 *    streams (and threads) are safe.
 *  - Range checks of input VALUES (residue < q_j, share < 2^t_bits) cost bandwidth and run
 *    only when the environment variable SECN_VALIDATE=1 is set when the context is created
 *    (then each call synchronises its stream and returns SECN_ERANGE on a violation; validated
 *    calls on one context are serialised, and they cannot be captured into a CUDA graph).
 *  - The other SECN_* environment variables are developer tuning knobs, also read once at
 *    context creation; the defaults are the measured best.
 *  - Ordering: a call may be scheduled, through programmatic dependent launch, while the
 *    preceding kernel on `stream` finishes; it reads nothing that kernel may have written before
 *    waiting for it, so inputs written by any earlier work on the stream are always seen.
 *  - Tracing: every call that enqueues work opens an NVTX range named after the entry point
 *    (nsys / ncu --nvtx group its kernels under it; a no-op when no tool is attached).
 */
#ifndef SECN_H_
#define SECN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SECN_MAX_LIMBS 4

typedef struct secn_ctx secn_ctx; /* opaque */

typedef enum {
  SECN_OK = 0,
  SECN_EINVAL = -1,       /* NULL pointer, size/shape/plan inconsistency            */
  SECN_EUNSUPPORTED = -2, /* parameter outside the supported set (see each call)     */
  SECN_ERANGE = -3,       /* input value out of range (only with SECN_VALIDATE=1)    */
  SECN_ENOMEM = -4,       /* device allocation failed (ctx creation only)            */
  SECN_ECUDA = -5,        /* a CUDA runtime call failed (message has the CUDA error) */
  SECN_ESTATE = -6        /* context/device mismatch                                 */
} secn_status;

/* Packing plan for one convolution layer (reading R6-R8; Cheetah packing PAPER.md:131 §2.3,
 * :374 §6.1). Inputs: C,H,W,M,kh,kw,stride,pad (and optionally Hw,Ww). secn_conv_plan fills
 * the rest:
 *   OH,OW   output extent;  decim = 1 for a 1x1 kernel with stride > 1 (input pre-decimated);
 *           decim = 2: polyphase packing of a strided kernel larger than 1x1 (reading R7b): the
 *           window math below uses Ce = C s^2 phase channels Xe[(c s + u) s + v, i, j] =
 *           Xpad[c, i s + u, j s + v] and the kernel extent khe x kwe = ceil(kh/s) x ceil(kw/s)
 *           in place of C, kh, kw, and sh = 1 (every window position is an output). As an input
 *           with explicit Hw, Ww, decim = 2 requests that packing.
 *   Hp,Wp   extent of the effective (padded, decimated or phase-split) input the windows tile
 *   Cw,Hw,Ww window: Cw channels x Hw rows x Ww cols per polynomial, Cw*Hw*Ww <= N
 *   G = ceil(C/Cw) input channel groups; S = nbh*nbw spatial blocks
 *   O = (Cw-1)*Hw*Ww + (kh-1)*Ww + (kw-1), the offset of the first designated coefficient
 * Input poly (g,s): coeff[c*Hw*Ww + i*Ww + j] = Xe[g*Cw+c, h0+i, w0+j], (h0,w0) =
 * (bh*(Hw-kh+1), bw*(Ww-kw+1)), s = bh*nbw+bw. Kernel poly (m,g):
 * coeff[O - c*Hw*Ww - l*Ww - l'] = K[m, g*Cw+c, l, l']. Output (m,oy,ox) is coefficient
 * O + i*Ww + j of output ct (m,s) where (bh*(Hw-kh+1)+i, bw*(Ww-kw+1)+j) = (oy*sh, ox*sh),
 * sh = stride (1 if decim). */
typedef struct {
  uint32_t C, H, W, M, kh, kw, stride, pad; /* layer geometry (caller)                   */
  uint32_t Hw, Ww;                          /* 0 = choose (secn_conv_plan_ex rule); else validated */
  uint32_t OH, OW, decim, Hp, Wp;           /* filled (decim = 2 also an input, see above) */
  uint32_t Cw, G, S, nbh, nbw, O;           /* filled                                      */
  uint32_t s_begin, s_count;                /* output spatial-block slice (caller; 0, 0 = all S) */
} secn_conv_plan_t;
/* Slices of one layer's output (the multi-GPU partition). M may be a slice of the
 * output channels: pass a plan copy with M = the slice size and pointers offset to its weights,
 * mask rows, output ciphertexts and share rows. s_begin, s_count select the spatial blocks
 * [s_begin, s_begin + s_count) of S: the call computes only the output ciphertexts (m, s) with s in
 * that range, at their usual positions m*S + s of ct_out / r (which keep all S rows; the other rows
 * are neither read nor written), and writes y0 only at the outputs those blocks designate. The
 * input ciphertexts are always all G*S. s_count = 0 means all of S (then s_begin must be 0). */

typedef struct {
  uint32_t log_n, n, n_limbs, t_bits;
  uint64_t primes[SECN_MAX_LIMBS];
  uint64_t psi[SECN_MAX_LIMBS]; /* minimal primitive 2N-th roots (reading R4)              */
  int device;
  uint32_t word_bits; /* 64: secn_* residue calls (uint64 words); 32: secn32_* calls (uint32)    */
} secn_ctx_info;

/* Creates a context on CUDA device `device`: copies the primes, finds psi_j, and builds the
 * device tables (psi^brv(i) and psi^-brv(i) with Shoup companions, N^-1, floor(Q/t) mod q_j,
 * Q mod t). Supported: 12 <= log_n <= 15, 1 <= n_limbs <= 4, every prime q_j < 2^61 with
 * q_j = 1 (mod 2N) (probable-prime tested), distinct; 1 <= t_bits <= 44.
 * log_n = 15 (the NTT sweep's largest ring) serves the NTT / mask / share
 * calls only: secn_preprocess_weights and the secn_he_conv2d family return SECN_EUNSUPPORTED
 * for it. Returns SECN_EUNSUPPORTED otherwise, SECN_ENOMEM / SECN_ECUDA on device failure. */
int secn_ctx_create(secn_ctx** out, int device, uint32_t log_n, uint32_t n_limbs, const uint64_t* primes,
                    uint32_t t_bits);
int secn_ctx_destroy(secn_ctx* ctx);
int secn_ctx_query(const secn_ctx* ctx, secn_ctx_info* info);
const char* secn_last_error(void);

/* Host only. Fills `p` from its geometry for ring degree 2^log_n (or validates the caller's
 * Hw,Ww when both are nonzero), choosing the packing window by `rule`:
 *   SECN_PLAN_BYTES: the byte-min rule of reading R6 (the oracle's plan_conv);
 *   SECN_PLAN_TIME:  reading R6b, the modelled device time of the integer-issue-bound path
 *                    (output, MAC and input limb-polys plus bytes), G <= 30
 *                    (G <= 32 when no window has G <= 30).
 * The packing (and so the oracle's result for the same window) is exact for every window; the
 * rule only picks the fastest. coef_words64 = 8-byte words per coefficient of one ciphertext
 * component (L for 64-bit limbs, L/2 for 32-bit limbs). SECN_EUNSUPPORTED if no window fits
 * (kh*kw > N or Hp < kh), SECN_EINVAL for an unknown rule. */
#define SECN_PLAN_BYTES 0u
#define SECN_PLAN_TIME 1u
int secn_conv_plan_ex(uint32_t log_n, uint32_t coef_words64, uint32_t rule, secn_conv_plan_t* p);
/* secn_conv_plan_ex with SECN_PLAN_TIME (the default the bench and the Python binding use). */
int secn_conv_plan(uint32_t log_n, uint32_t coef_words64, secn_conv_plan_t* p);

/* A1: in-place forward negacyclic NTT of n_polys polys [n_polys][L][N] (coefficient domain ->
 * NTT domain), PAPER.md:378-380 (§6.2), App. C.1. At N = 2^15 (and 64-bit words at 2^14) each
 * limb-poly is transformed by a cluster of two CTAs (cluster NTT). */
int secn_ntt_fwd(secn_ctx* ctx, uint64_t* polys, size_t n_polys, void* stream);

/* A2: in-place inverse of secn_ntt_fwd, N^-1 included. */
int secn_ntt_inv(secn_ctx* ctx, uint64_t* polys, size_t n_polys, void* stream);

/* A3: NTT preprocessing of the weights (PAPER.md:376-380 §6.2, :427 §7 step 1, :445 §8.1):
 * kernel [M][C][kh][kw] (values < 2^t_bits, two's complement mod 2^t) is packed into the
 * mirrored plaintext polys of `plan`, centred-lifted to every q_j (reading R3) and transformed:
 * w_ntt [M][G][L][N] (NTT domain). Deterministic (idempotent). Uses only `plan->M` kernels. */
int secn_preprocess_weights(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* kernel, uint64_t* w_ntt,
                            void* stream);

/* A6: server-share add (§7): for ct [n][2][L][N] (coefficient domain),
 * b_j += enc_j(x0) with x0 [n][N] < 2^t_bits. */
int secn_share_add(secn_ctx* ctx, uint64_t* ct, const uint64_t* x0, size_t n, void* stream);

/* A7: random output mask (§7): b_j += enc_j(r) for ct [n][2][L][N]
 * (coefficient domain), r [n][N] < 2^t_bits. The server's share is (t - r) mod t. */
int secn_mask_add(secn_ctx* ctx, uint64_t* ct, const uint64_t* r, size_t n, void* stream);

/* Bytes of device workspace the secn_he_conv2d family needs for `plan`: the NTT-domain inputs
 * X^ = G*S*2*L*N words of the context's word size (all a call with a caller mask r or a
 * pre-encoded mask needs), then the encoded mask (M*S*L*N words) for the *_gen calls. */
size_t secn_he_conv2d_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan);

/* The hot path (PAPER.md:380 §6.2, :431 §7), one layer:
 *   in'  = ct_in with b += enc(x0)                       (A6, fused; skipped if x0 == NULL)
 *   X^   = NTT(in')                                       (A1)
 *   Y^[m,s] = sum_{g<G} X^[g,s] (.) w_ntt[m,g]            (A4, both components, every limb)
 *   out  = INTT(Y^), then b += enc(r[m,s])                (A2 + A7 fused; skipped if r == NULL)
 * ct_in [G*S][2][L][N] coefficient domain (index g*S+s) -- read only;
 * x0 [G*S][N] or NULL; w_ntt [M][G][L][N] from secn_preprocess_weights (M = plan->M, which may
 * be a slice of the layer's output channels: pass a plan copy with M = slice size and
 * pointers offset to the slice); r [M*S][N] or NULL; ct_out [M*S][2][L][N] (index m*S+s,
 * coefficient domain, overwritten; must not alias the inputs); workspace >=
 * secn_he_conv2d_workspace bytes, 16-byte aligned. */
int secn_he_conv2d(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                   const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, void* workspace, size_t ws_bytes,
                   void* stream);

/* The same computation as secn_he_conv2d, one launch group at a time, so a caller can time
 * each kernel with events on `stream`: stage 0 = A6+A1 (ct_in, x0 -> workspace X^),
 * stage 1 = A4 and the first 8 inverse-NTT levels (workspace, w_ntt -> ct_out holding Y^ after
 * Gentleman-Sande levels 0..7, values in the lazy range [0, 2q) / [0, 4q)), stage 2 = the
 * remaining inverse-NTT levels, N^-1 and A7 (ct_out in place, r). Running stages 0,1,2 in order
 * on one stream equals secn_he_conv2d; only the final ct_out is canonical.
 * Arguments as for secn_he_conv2d; SECN_EINVAL for any other `stage`. */
int secn_he_conv2d_stage(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint64_t* ct_in,
                         const uint64_t* x0, const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out,
                         void* workspace, size_t ws_bytes, void* stream);

/* secn_he_conv2d plus the server's output share (A8, as secn_extract_share) in the same
 * launches: y0 [M][OH][OW] (uint64, < 2^t_bits) is written from r by the inverse-NTT tail
 * kernel. y0 may be NULL (then identical to secn_he_conv2d); y0 != NULL needs r != NULL
 * (else SECN_EINVAL). y0 must not alias any other argument. */
int secn_he_conv2d_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                      const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
                      size_t ws_bytes, void* stream);

/* Online NTT preprocessing ("linear layers with
 * online/offline/no NTT preprocessing"): the same result as secn_preprocess_weights followed by
 * secn_he_conv2d_ex, in one call, with the kernel in coefficient form ([M][C][kh][kw] uint64
 * < 2^t_bits, as for secn_preprocess_weights). The transformed weights live in the workspace
 * (>= secn_he_conv2d_online_workspace bytes, 16-byte aligned), so nothing query-independent
 * is kept between calls: the server trades the weight bytes it would hold for an NTT per query.
 * y0 may be NULL. Errors as for secn_preprocess_weights and secn_he_conv2d_ex. */
size_t secn_he_conv2d_online_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan);
int secn_he_conv2d_online(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                          const uint64_t* kernel, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
                          size_t ws_bytes, void* stream);

/* Server's output share at the designated coefficients (§7; Cheetah's sparse
 * result): y0[m][oy][ox] = (t - r[m*S+s][O + i*Ww + j]) mod t for the plan's
 * index map, m in [0, plan->M). r [M*S][N], y0 [M][OH][OW]. */
int secn_extract_share(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* r, uint64_t* y0, void* stream);

/* ------------------------------------------------------------------------------------------
 * Device-drawn mask (§7, "applies a random mask for security"; reading R17).
 * The calls above take the server's mask r from the caller. These draw it on the device from the
 * counter-based generator Philox4x32-10 (Salmon et al., SC'11), so the server's own randomness
 * never crosses PCIe:
 *   (w0, w1, w2, w3) = Philox4x32-10(counter = (e >> 1, ct0 + c, stream, 0),
 *                                    key = (seed mod 2^32, seed >> 32))
 *   r[c][e] = (w1 2^32 + w0) mod 2^t_bits for even e,  (w3 2^32 + w2) mod 2^t_bits for odd e,
 * for output ciphertext c of the call (the layer's index m*S + s; ct0 lets a rank slice of the
 * output channels draw exactly the rows of the whole layer it owns) and coefficient e. A fresh
 * (seed, stream) per query and layer is the caller's responsibility.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  uint64_t seed;   /* generator key                                                           */
  uint32_t stream; /* e.g. (query, layer) id: distinct streams give independent masks          */
  uint32_t ct0;    /* index of the call's first output ciphertext in the layer (0 = whole layer) */
} secn_mask_gen_t;

/* r [n_ct][N] (uint64 < 2^t_bits, device, 16-byte aligned) for output ciphertexts ct0 .. ct0+n_ct-1.
 * SECN_EINVAL for a NULL generator or buffer. */
int secn_mask_draw(secn_ctx* ctx, const secn_mask_gen_t* gen, size_t n_ct, uint64_t* r, void* stream);

/* secn_he_conv2d_ex with r drawn by `gen` (the draw runs between the forward NTT and the MAC and
 * lands in the workspace, >= secn_he_conv2d_gen_workspace bytes). y0 (may be NULL) receives the
 * server's share -r mod t at the designated coefficients, as with a caller-supplied r. */
size_t secn_he_conv2d_gen_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan);
int secn_he_conv2d_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                       const uint64_t* w_ntt, const secn_mask_gen_t* gen, uint64_t* ct_out, uint64_t* y0,
                       void* workspace, size_t ws_bytes, void* stream);

/* The encoded mask, prepared apart from the layer call. The mask is input-independent, so a server
 * can draw and encode it ahead of (or concurrently with) the computation that needs it, e.g. on a
 * low-priority stream while earlier layers run (bench.py does). secn_mask_encode writes
 * em [M*S][L][N] (words of the context's size, secn_mask_encoded_bytes bytes, 16-byte aligned):
 * em[m*S + s][j][e] = enc_j(r[m*S + s][e]) for the plan's output ciphertexts (its spatial slice;
 * M may be a channel slice as elsewhere) with r from the caller (r [M*S][N] < 2^t_bits) or drawn
 * by `gen` (exactly one of r, gen), and y0 (may be NULL) = -r mod t at the designated outputs.
 * secn_he_conv2d_em / secn32_he_conv2d_em then run the layer adding em (A7) -- the result of
 * secn_he_conv2d_ex with that r. The LWE form is secn[32]_he_conv2d_lwe_em. */
size_t secn_mask_encoded_bytes(const secn_ctx* ctx, const secn_conv_plan_t* plan);
int secn_mask_encode(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* r, const secn_mask_gen_t* gen,
                     void* em, uint64_t* y0, void* stream);
int secn_he_conv2d_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                      const uint64_t* w_ntt, const uint64_t* em, uint64_t* ct_out, void* workspace, size_t ws_bytes,
                      void* stream);

/* ------------------------------------------------------------------------------------------
 * HE fully-connected layer / matrix-vector product (§6
 * "fully-connected/matrix multiplication layers"; SPEC.md:612-619 fc_secure). The server's work
 * is the convolution's -- share add + NTT of the input cts, NTT-domain MAC over input blocks,
 * inverse NTT + mask -- with the matrix-vector packing of DESIGN.md reading R15:
 *   input ct g:           coeff[i]                   = x[g*nib + i]                 (i < nib)
 *   weight poly (m, g):   coeff[j*nib + nib - 1 - i] = W[m*nob + j][g*nib + i]      (j < nob)
 *   output ct m holds y[m*nob + j] at coefficient j*nib + nib - 1.
 * ------------------------------------------------------------------------------------------ */
typedef struct {
  uint32_t n_i, n_o; /* matrix W: n_o rows x n_i columns (caller)                                */
  uint32_t nib;      /* input values per ct: 0 = choose (byte-min rule R15); else validated      */
  uint32_t nob;      /* filled: output rows per ct = min(n_o, N / nib)                            */
  uint32_t G, M;     /* filled: input cts ceil(n_i/nib), output cts ceil(n_o/nob)                 */
} secn_fc_plan_t;

/* Host only: fills nob, G, M (and nib when 0) for ring degree 2^log_n; coef_words64 as for
 * secn_conv_plan. SECN_EINVAL for n_i or n_o = 0 or an invalid nib (0 < nib <= min(n_i, N)). */
int secn_fc_plan(uint32_t log_n, uint32_t coef_words64, secn_fc_plan_t* p);

/* Offline NTT preprocessing of the matrix: W [n_o][n_i] uint64 (< 2^t_bits, two's complement
 * mod 2^t) -> w_ntt [M][G][L][N] (NTT domain, centred lift per limb, reading R3). */
int secn_fc_preprocess_weights(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* W, uint64_t* w_ntt,
                               void* stream);

/* Workspace bytes for secn_he_fc (the NTT-domain inputs, G*2*L*N words). */
size_t secn_he_fc_workspace(const secn_ctx* ctx, const secn_fc_plan_t* plan);

/* One FC layer: ct_in [G][2][L][N] (coefficient domain, read only), x0 [G][N] or NULL (the
 * server's input share, packed like x), w_ntt from secn_fc_preprocess_weights, r [M][N] or NULL,
 * ct_out [M][2][L][N] (overwritten), y0 [n_o] or NULL (needs r): the server's output share
 * (t - r[m][j*nib + nib - 1]) mod t. SECN_EUNSUPPORTED if G > 32 or log_n > 14. */
int secn_he_fc(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
               const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
               size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * Extracted outputs (Cheetah's sparse result PAPER.md:131 §2.3; the result
 * returned to the client PAPER.md:431 §7; reading R16). The same computation as
 * secn_he_conv2d_ex / secn_he_fc, but each output ciphertext leaves the kernel
 *   (1) switched to the first keep_limbs primes Q' = q_0..q_{keep-1}: every coefficient c (both
 *       components) becomes round(c Q'/Q) mod Q' (exact, RNS, no ties since Q/Q' is odd);
 *   (2) extracted: the a component whole, a_out [n_ct][keep][N]; the b component only at its
 *       designated coefficients, b_out [value][keep] with value = (m, oy, ox) row-major for a
 *       convolution ([M][OH][OW]) and the output row o for a matrix-vector product ([n_o]).
 * The client decrypts value k of ct n as round(t (b'_k - (a'_n * sk)_k) / Q') mod t (an LWE
 * decryption). y0 as for secn_he_conv2d_ex. N = 4096 only; keep_limbs in [1, L-1] with the
 * dropped primes' product < 2^62 (SECN_EUNSUPPORTED otherwise; Q'/t must leave room for the
 * switching noise: keep 2 of 4 27-bit limbs, or 1 of the 60+49-bit pair). The workspace holds
 * X^ and the output cts before switching (secn_he_*_lwe_workspace bytes). */
size_t secn_he_conv2d_lwe_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan);
int secn_he_conv2d_lwe(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                       const uint64_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint64_t* a_out,
                       uint64_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);
/* secn_he_conv2d_lwe with the mask drawn by `gen` (reading R17; workspace >=
 * secn_he_conv2d_lwe_gen_workspace bytes). */
size_t secn_he_conv2d_lwe_gen_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan);
int secn_he_conv2d_lwe_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                           const uint64_t* w_ntt, const secn_mask_gen_t* gen, uint32_t keep_limbs, uint64_t* a_out,
                           uint64_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);
int secn_he_conv2d_lwe_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                          const uint64_t* w_ntt, const uint64_t* em, uint32_t keep_limbs, uint64_t* a_out,
                          uint64_t* b_out, void* workspace, size_t ws_bytes, void* stream);
size_t secn_he_fc_lwe_workspace(const secn_ctx* ctx, const secn_fc_plan_t* plan);
int secn_he_fc_lwe(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                   const uint64_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint64_t* a_out, uint64_t* b_out,
                   uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------------------------
 * 32-bit RNS limbs (reading R1b). Identical semantics to the
 * calls above with residues stored as uint32 ([..][L][N] uint32 words) for moduli q_j < 2^28,
 * e.g. four 27-bit primes = 1 mod 2^16 (Q = 108 bits <= 109, the 128-bit-security bound for
 * N = 4096). The same bytes per coefficient as two 64-bit limbs, but every modular product is a
 * 32x32-bit Shoup/IMAD.WIDE operation. Plaintext-side arrays (x0, r, kernels, y0) stay uint64.
 * A 32-bit context rejects the 64-bit residue calls (and vice versa) with SECN_ESTATE;
 * secn_ctx_destroy/query, secn_conv_plan, secn_he_conv2d_workspace (bytes for the context's word
 * size) and secn_extract_share serve both.
 * ------------------------------------------------------------------------------------------ */
int secn32_ctx_create(secn_ctx** out, int device, uint32_t log_n, uint32_t n_limbs, const uint32_t* primes,
                      uint32_t t_bits);
int secn32_ntt_fwd(secn_ctx* ctx, uint32_t* polys, size_t n_polys, void* stream);
int secn32_ntt_inv(secn_ctx* ctx, uint32_t* polys, size_t n_polys, void* stream);
int secn32_preprocess_weights(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* kernel, uint32_t* w_ntt,
                              void* stream);
int secn32_share_add(secn_ctx* ctx, uint32_t* ct, const uint64_t* x0, size_t n, void* stream);
int secn32_mask_add(secn_ctx* ctx, uint32_t* ct, const uint64_t* r, size_t n, void* stream);
int secn32_he_conv2d(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                     const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, void* workspace, size_t ws_bytes,
                     void* stream);
int secn32_he_conv2d_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                        const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, uint64_t* y0, void* workspace,
                        size_t ws_bytes, void* stream);
int secn32_he_conv2d_online(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                            const uint64_t* kernel, const uint64_t* r, uint32_t* ct_out, uint64_t* y0,
                            void* workspace, size_t ws_bytes, void* stream);
int secn32_fc_preprocess_weights(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* W, uint32_t* w_ntt,
                                 void* stream);
int secn32_he_fc(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                 const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, uint64_t* y0, void* workspace,
                 size_t ws_bytes, void* stream);
int secn32_he_conv2d_lwe(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                         const uint32_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint32_t* a_out,
                         uint32_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);
int secn32_he_fc_lwe(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                     const uint32_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint32_t* a_out, uint32_t* b_out,
                     uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);
int secn32_he_conv2d_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                         const uint32_t* w_ntt, const secn_mask_gen_t* gen, uint32_t* ct_out, uint64_t* y0,
                         void* workspace, size_t ws_bytes, void* stream);
int secn32_he_conv2d_lwe_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                             const uint32_t* w_ntt, const secn_mask_gen_t* gen, uint32_t keep_limbs, uint32_t* a_out,
                             uint32_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);
int secn32_he_conv2d_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                        const uint32_t* w_ntt, const uint32_t* em, uint32_t* ct_out, void* workspace, size_t ws_bytes,
                        void* stream);
int secn32_he_conv2d_lwe_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                            const uint32_t* w_ntt, const uint32_t* em, uint32_t keep_limbs, uint32_t* a_out,
                            uint32_t* b_out, void* workspace, size_t ws_bytes, void* stream);
int secn32_he_conv2d_stage(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint32_t* ct_in,
                           const uint64_t* x0, const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out,
                           void* workspace, size_t ws_bytes, void* stream);
/* secn_he_conv2d_stage with the server's output share: y0 (as in secn_he_conv2d_ex; may be NULL)
 * is written by stage 2 (the kernel that also adds the mask), which is where the fused call
 * writes it; stages 0 and 1 ignore y0. Lets a caller overlap one launch group of several
 * independent layers at a time (bench.py --overlap staged). */
int secn_he_conv2d_stage_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint64_t* ct_in,
                            const uint64_t* x0, const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0,
                            void* workspace, size_t ws_bytes, void* stream);
int secn32_he_conv2d_stage_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint32_t* ct_in,
                              const uint64_t* x0, const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out,
                              uint64_t* y0, void* workspace, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SECN_H_ */
