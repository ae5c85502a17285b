// libsecn host side: the C ABI declared in include/secn.h -- context/table construction,
// packing plan, argument validation and kernel dispatch. No torch types anywhere.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

#include <nvtx3/nvToolsExt.h>

typedef unsigned __int128 u128;

namespace {

thread_local std::string g_err;

// An NVTX range named after the entry point around every call that launches work (nsys/ncu
// --nvtx timelines group the call's kernels under it; without a tool attached, a no-op).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SECN_NVTX() NvtxRange secn_nvtx_range_(__func__)

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(SECN_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ---- 64-bit number theory with 128-bit intermediates (host) ----
uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)((u128)a * b % q); }

uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  for (; e; e >>= 1) {
    if (e & 1) r = mulmod(r, b, q);
    b = mulmod(b, b, q);
  }
  return r;
}

bool probable_prime(uint64_t n) {
  if (n < 2) return false;
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t p : bases)
    if (n % p == 0) return n == p;
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (uint64_t a : bases) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s && comp; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}

uint64_t shoup_companion(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

uint32_t bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
  return r;
}

// The smallest primitive 2N-th root of unity mod prime q (reading R4): psi^N = -1; the
// primitive 2N-th roots are the odd powers of any one of them.
uint64_t min_primitive_root(uint64_t q, uint64_t n) {
  for (uint64_t x = 2; x < q; ++x) {
    const uint64_t y = powmod(x, (q - 1) / (2 * n), q);
    if (powmod(y, n, q) != q - 1) continue;
    const uint64_t y2 = mulmod(y, y, q);
    uint64_t best = y, cur = y;
    for (uint64_t k = 3; k < 2 * n; k += 2) {
      cur = mulmod(cur, y2, q);
      if (cur < best) best = cur;
    }
    return best;
  }
  return 0;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// With SECN_VALIDATE=1 (read at context creation): synchronously check that `n_words` words are
// in range (kind 0: residues < q_j by limb, kind 1: < 2^t_bits). The context's one flag word is
// shared by every validated call, so the whole check runs under the context's mutex.
int check_range(secn_ctx* ctx, const void* v, size_t n_words, int kind, cudaStream_t s, const char* what) {
  if (!ctx->dc.tune.validate || v == nullptr || n_words == 0) return SECN_OK;
  std::lock_guard<std::mutex> lock(*ctx->flag_mutex);
  cudaError_t e = cudaMemsetAsync(ctx->d_flag, 0, sizeof(uint32_t), s);
  if (e == cudaSuccess) e = secn::launch_check_range(ctx->dc, v, n_words, kind, ctx->d_flag, s);
  uint32_t flag = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, ctx->d_flag, sizeof flag, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "range check");
  if (flag) return fail(SECN_ERANGE, "%s: value out of range (%s)", what, kind == 0 ? ">= q_j" : ">= 2^t_bits");
  return SECN_OK;
}

// polyphase factor of a plan (reading R7b): the stride when decim = 2, else 1
uint32_t plan_ps(const secn_conv_plan_t* p) { return p->decim == 2 ? p->stride : 1; }

secn::PlanDev plan_dev(const secn_conv_plan_t* p) {
  secn::PlanDev d{};
  const uint32_t ps = plan_ps(p);
  d.M = p->M, d.G = p->G, d.S = p->S, d.Cw = p->Cw, d.Hw = p->Hw, d.Ww = p->Ww;
  d.kh = (p->kh + ps - 1) / ps, d.kw = (p->kw + ps - 1) / ps;  // the window's kernel extent
  d.kh0 = p->kh, d.kw0 = p->kw, d.ps = ps;                      // the caller's kernel tensor
  d.C = p->C, d.O = p->O, d.OH = p->OH, d.OW = p->OW, d.nbh = p->nbh, d.nbw = p->nbw;
  d.sh = p->decim ? 1 : p->stride;
  d.s0 = p->s_count ? p->s_begin : 0, d.sn = p->s_count ? p->s_count : p->S;
  return d;
}

// Recompute the derived fields of a plan from its geometry, (Hw, Ww) and the polyphase choice
// (reading R7b, strided kernels larger than 1x1 only); 0 if consistent.
int derive_plan(uint32_t n, uint32_t Hw, uint32_t Ww, bool poly, secn_conv_plan_t* p) {
  const uint32_t C = p->C, kh = p->kh, kw = p->kw, st = p->stride, pad = p->pad;
  if (!C || !p->H || !p->W || !p->M || !kh || !kw || !st) return -1;
  if (p->H + 2 * pad < kh || p->W + 2 * pad < kw) return -1;
  const uint32_t OH = (p->H + 2 * pad - kh) / st + 1, OW = (p->W + 2 * pad - kw) / st + 1;
  uint32_t decim = (kh == 1 && kw == 1 && st > 1) ? 1 : 0;
  if (poly) {
    if (decim || st == 1) return -1;
    decim = 2;
  }
  uint32_t Hp, Wp, Ph, Pw;
  if (decim == 1) {
    Hp = Ph = OH, Wp = Pw = OW;
  } else if (decim == 2) {
    Hp = (p->H + 2 * pad + st - 1) / st, Wp = (p->W + 2 * pad + st - 1) / st, Ph = OH, Pw = OW;
  } else {
    Hp = p->H + 2 * pad, Wp = p->W + 2 * pad, Ph = (OH - 1) * st + 1, Pw = (OW - 1) * st + 1;
  }
  const uint32_t ps = decim == 2 ? st : 1, Ce = C * ps * ps, khe = (kh + ps - 1) / ps, kwe = (kw + ps - 1) / ps;
  if (Hw < khe || Ww < kwe || Hw > Hp || Ww > Wp || (uint64_t)Hw * Ww > n) return -1;
  const uint32_t Cw = Ce < n / (Hw * Ww) ? Ce : n / (Hw * Ww);
  p->OH = OH, p->OW = OW, p->decim = decim, p->Hp = Hp, p->Wp = Wp, p->Hw = Hw, p->Ww = Ww, p->Cw = Cw;
  p->G = (Ce + Cw - 1) / Cw;
  p->nbh = (Ph + (Hw - khe)) / (Hw - khe + 1);
  p->nbw = (Pw + (Ww - kwe)) / (Ww - kwe + 1);
  p->S = p->nbh * p->nbw;
  p->O = (Cw - 1) * Hw * Ww + (khe - 1) * Ww + (kwe - 1);
  return 0;
}

int check_ctx(const secn_ctx* ctx, uint32_t want_bits = 0) {
  if (!ctx) return fail(SECN_EINVAL, "NULL context");
  if (want_bits && ctx->word_bits != want_bits)
    return fail(SECN_ESTATE, "context has %u-bit residues; use the secn%s_ entry points", ctx->word_bits,
                ctx->word_bits == 32 ? "32" : "");
  int dev;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SECN_ESTATE, "no current CUDA device");
  return SECN_OK;
}

int check_plan(const secn_ctx* ctx, const secn_conv_plan_t* p) {
  if (!p) return fail(SECN_EINVAL, "NULL plan");
  secn_conv_plan_t q = *p;
  if (derive_plan(ctx->n, p->Hw, p->Ww, p->decim == 2, &q) != 0)
    return fail(SECN_EINVAL, "plan inconsistent with its geometry");
  if (q.Cw != p->Cw || q.G != p->G || q.S != p->S || q.O != p->O || q.OH != p->OH || q.OW != p->OW ||
      q.decim != p->decim || q.nbh != p->nbh || q.nbw != p->nbw)
    return fail(SECN_EINVAL, "plan fields do not match secn_conv_plan() for this geometry and N");
  if (p->s_count ? (uint64_t)p->s_begin + p->s_count > p->S : p->s_begin != 0)
    return fail(SECN_EINVAL, "spatial slice [%u, %u + %u) not inside S = %u", p->s_begin, p->s_begin, p->s_count, p->S);
  return SECN_OK;
}

}  // namespace

extern "C" {

const char* secn_last_error(void) { return g_err.c_str(); }

static int ctx_create_impl(secn_ctx** out, int device, uint32_t log_n, uint32_t n_limbs, const uint64_t* primes,
                           uint32_t t_bits, uint32_t word_bits) {
  if (!out || !primes) return fail(SECN_EINVAL, "NULL argument");
  *out = nullptr;
  if (log_n < 12 || log_n > 15) return fail(SECN_EUNSUPPORTED, "log_n=%u not in [12,15]", log_n);
  if (n_limbs < 1 || n_limbs > SECN_MAX_LIMBS) return fail(SECN_EUNSUPPORTED, "n_limbs=%u not in [1,4]", n_limbs);
  if (t_bits < 1 || t_bits > 44) return fail(SECN_EUNSUPPORTED, "t_bits=%u not in [1,44]", t_bits);
  const uint64_t n = 1ull << log_n;
  const uint64_t qmax = word_bits == 64 ? (1ull << 61) : (1ull << 28);
  for (uint32_t j = 0; j < n_limbs; ++j) {
    const uint64_t q = primes[j];
    if (q >= qmax) return fail(SECN_EUNSUPPORTED, "prime %u >= 2^%d", j, word_bits == 64 ? 61 : 28);
    if (word_bits == 64 && q <= (1ull << t_bits)) return fail(SECN_EUNSUPPORTED, "prime %u <= 2^t_bits", j);
    if ((q - 1) % (2 * n) != 0) return fail(SECN_EUNSUPPORTED, "prime %u != 1 mod 2N", j);
    if (!probable_prime(q)) return fail(SECN_EUNSUPPORTED, "modulus %u is not prime", j);
    for (uint32_t k = 0; k < j; ++k)
      if (primes[k] == q) return fail(SECN_EUNSUPPORTED, "duplicate prime");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(SECN_ESTATE, "device %d not available", device);
  DeviceGuard guard(device);
  if (cudaError_t e = secn::init_device(word_bits); e != cudaSuccess) return cuda_fail(e, "kernel attributes");

  secn_ctx* c = new secn_ctx();
  c->device = device, c->log_n = log_n, c->n = (uint32_t)n, c->L = n_limbs, c->t_bits = t_bits;
  c->word_bits = word_bits;
  secn::DevConsts& dc = c->dc;
  std::memset(&dc, 0, sizeof dc);
  dc.t_bits = t_bits, dc.log_n = log_n, dc.L = n_limbs, dc.word_bits = word_bits;
  secn::read_tune(device, &dc.tune);
  const uint64_t t = 1ull << t_bits, tmask = t - 1;
  // Q mod t = prod (q_j mod t) mod t (t a power of two)
  uint64_t qmt = 1;
  for (uint32_t j = 0; j < n_limbs; ++j) qmt = (uint64_t)(((u128)qmt * (primes[j] & tmask)) & tmask);
  dc.qmt = qmt;
  // Shoup companion over the word size
  auto comp = [&](uint64_t w, uint64_t q) {
    return word_bits == 64 ? shoup_companion(w, q) : (uint64_t)((((u128)w) << 32) / q);
  };
  // full tables [2][L][N] (fwd, inv); for the cluster NTT (N = 2^15, or 64-bit words at 2^14)
  // also the per-half tables [2][L][2][N/2]
  const bool halves = log_n == 15 || (log_n == 14 && word_bits == 64);
  const size_t tw_bytes = (word_bits == 64 ? sizeof(ulonglong2) : sizeof(uint2)) * 2 * n_limbs * n * (halves ? 2 : 1);
  std::vector<unsigned char> tw(tw_bytes);
  ulonglong2* tw64 = reinterpret_cast<ulonglong2*>(tw.data());
  uint2* tw32 = reinterpret_cast<uint2*>(tw.data());
  bool redc = word_bits == 32;  // k_mac's Montgomery REDC needs G q < 2^32 for G <= 32: q < 2^27
  for (uint32_t j = 0; j < n_limbs; ++j) redc = redc && primes[j] < (1ull << 27);
  dc.mac_redc = redc ? 1u : 0u;
  for (uint32_t j = 0; j < n_limbs; ++j) {
    const uint64_t q = primes[j];
    c->primes[j] = q;
    const uint64_t psi = min_primitive_root(q, n);
    c->psi[j] = psi;
    const uint64_t psi_inv = powmod(psi, q - 2, q);
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t e = bitrev(i, log_n);
      const uint64_t wf = powmod(psi, e, q), wi = powmod(psi_inv, e, q);
      const size_t fi = (size_t)j * n + i, ii = ((size_t)n_limbs + j) * n + i;
      if (word_bits == 64) {
        tw64[fi] = make_ulonglong2(wf, comp(wf, q));
        tw64[ii] = make_ulonglong2(wi, comp(wi, q));
      } else {
        tw32[fi] = make_uint2((uint32_t)wf, (uint32_t)comp(wf, q));
        tw32[ii] = make_uint2((uint32_t)wi, (uint32_t)comp(wi, q));
      }
    }
    dc.q[j] = q;
    const uint64_t ninv = powmod(n % q, q - 2, q);
    dc.ninv[j] = ninv, dc.ninv_p[j] = comp(ninv, q);
    const uint64_t wl = mulmod(powmod(psi_inv, bitrev(1, log_n), q), ninv, q);
    dc.wlast[j] = wl, dc.wlast_p[j] = comp(wl, q);
    {
      const uint64_t scale = redc ? (uint64_t)((((u128)1) << 32) % q) : 1;  // undoes REDC's 2^-32
      const uint64_t nm = mulmod(ninv, scale, q), wm = mulmod(wl, scale, q);
      dc.ninv_mac[j] = nm, dc.ninv_mac_p[j] = comp(nm, q);
      dc.wlast_mac[j] = wm, dc.wlast_mac_p[j] = comp(wm, q);
      uint32_t qi = 1;  // q^-1 mod 2^32 by Newton iteration (q odd)
      for (int it = 0; it < 5; ++it) qi *= 2u - (uint32_t)q * qi;
      dc.qneg_inv32[j] = (uint32_t)(0u - qi);
    }
    // floor(Q/t) = (Q - (Q mod t)) / t and Q = 0 mod q_j  =>  floor(Q/t) = -(Q mod t) t^-1 mod q_j
    const uint64_t tinv = powmod(t % q, q - 2, q);
    const uint64_t delta = mulmod((q - qmt % q) % q, tinv, q);
    dc.delta[j] = delta, dc.delta_p[j] = shoup_companion(delta, q);
    dc.tinv[j] = tinv, dc.tinv_p[j] = comp(tinv, q);
    const uint64_t tinv_hi = (uint64_t)((((u128)tinv) << 32) % q);
    dc.tinv_hi[j] = tinv_hi, dc.tinv_hi_p[j] = comp(tinv_hi, q);
    const uint64_t r32 = (uint64_t)((1ull << 32) % q);
    dc.r32[j] = r32, dc.r32_p[j] = word_bits == 32 ? (uint64_t)((((u128)r32) << 32) / q) : 0;
    const uint64_t r64 = (uint64_t)(((u128)1 << 64) % q);
    dc.r64[j] = r64, dc.r64_p[j] = shoup_companion(r64, q);
    dc.one_p[j] = ~0ull / q;
    dc.one_wp[j] = comp(1, q);
    if (halves) {  // half tables: th[k] = t[k + hp2(k) (1 + h)] (see DevConsts)
      const size_t nh = n / 2, base = 2 * (size_t)n_limbs * n;
      for (uint32_t h = 0; h < 2; ++h)
        for (uint32_t k = 0; k < nh; ++k) {
          uint32_t hp2 = 1;
          while (k && hp2 * 2 <= k) hp2 *= 2;
          const size_t src = k ? k + (size_t)hp2 * (1 + h) : 0;
          for (uint32_t dir = 0; dir < 2; ++dir) {
            const size_t from = ((size_t)dir * n_limbs + j) * n + src;
            const size_t to = base + (((size_t)dir * n_limbs + j) * 2 + h) * nh + k;
            if (word_bits == 64)
              tw64[to] = tw64[from];
            else
              tw32[to] = tw32[from];
          }
        }
    }
  }
  cudaError_t e = cudaMalloc(&c->d_tables, tw_bytes);
  if (e != cudaSuccess) {
    delete c;
    return fail(e == cudaErrorMemoryAllocation ? SECN_ENOMEM : SECN_ECUDA, "cudaMalloc tables: %s", cudaGetErrorString(e));
  }
  e = cudaMalloc(&c->d_flag, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemcpy(c->d_tables, tw.data(), tw_bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(c->d_tables);
    cudaFree(c->d_flag);
    delete c;
    return cuda_fail(e, "ctx tables");
  }
  c->flag_mutex = new std::mutex();
  if (word_bits == 64) {
    dc.tw_fwd = static_cast<const ulonglong2*>(c->d_tables);
    dc.tw_inv = dc.tw_fwd + (size_t)n_limbs * n;
    if (halves) dc.tw_fwd_h = dc.tw_fwd + 2 * (size_t)n_limbs * n, dc.tw_inv_h = dc.tw_fwd_h + (size_t)n_limbs * n;
  } else {
    dc.tw32_fwd = static_cast<const uint2*>(c->d_tables);
    dc.tw32_inv = dc.tw32_fwd + (size_t)n_limbs * n;
    if (halves)
      dc.tw32_fwd_h = dc.tw32_fwd + 2 * (size_t)n_limbs * n, dc.tw32_inv_h = dc.tw32_fwd_h + (size_t)n_limbs * n;
  }
  *out = c;
  return SECN_OK;
}

int secn_ctx_create(secn_ctx** out, int device, uint32_t log_n, uint32_t n_limbs, const uint64_t* primes,
                    uint32_t t_bits) {
  SECN_NVTX();
  return ctx_create_impl(out, device, log_n, n_limbs, primes, t_bits, 64);
}

int secn32_ctx_create(secn_ctx** out, int device, uint32_t log_n, uint32_t n_limbs, const uint32_t* primes,
                      uint32_t t_bits) {
  SECN_NVTX();
  if (!primes) return fail(SECN_EINVAL, "NULL argument");
  uint64_t p64[SECN_MAX_LIMBS] = {0, 0, 0, 0};
  for (uint32_t j = 0; j < n_limbs && j < SECN_MAX_LIMBS; ++j) p64[j] = primes[j];
  return ctx_create_impl(out, device, log_n, n_limbs, p64, t_bits, 32);
}

int secn_ctx_destroy(secn_ctx* ctx) {
  if (!ctx) return SECN_OK;
  DeviceGuard guard(ctx->device);
  cudaFree(ctx->d_tables);
  cudaFree(ctx->d_flag);
  delete ctx->flag_mutex;
  delete ctx;
  return SECN_OK;
}

int secn_ctx_query(const secn_ctx* ctx, secn_ctx_info* info) {
  if (!ctx || !info) return fail(SECN_EINVAL, "NULL argument");
  std::memset(info, 0, sizeof *info);
  info->log_n = ctx->log_n, info->n = ctx->n, info->n_limbs = ctx->L, info->t_bits = ctx->t_bits;
  info->device = ctx->device;
  info->word_bits = ctx->word_bits;
  for (uint32_t j = 0; j < ctx->L; ++j) info->primes[j] = ctx->primes[j], info->psi[j] = ctx->psi[j];
  return SECN_OK;
}

int secn_conv_plan_ex(uint32_t log_n, uint32_t n_limbs /* coef_words64 */, uint32_t rule, secn_conv_plan_t* p) {
  if (!p) return fail(SECN_EINVAL, "NULL plan");
  if (log_n < 1 || log_n > 20 || n_limbs < 1) return fail(SECN_EUNSUPPORTED, "bad log_n / n_limbs");
  if (rule > SECN_PLAN_TIME) return fail(SECN_EINVAL, "unknown plan rule %u", rule);
  const uint32_t n = 1u << log_n;
  if (!p->C || !p->H || !p->W || !p->M || !p->kh || !p->kw || !p->stride)
    return fail(SECN_EINVAL, "zero dimension in plan geometry");
  if ((uint64_t)p->kh * p->kw > n || p->H + 2 * p->pad < p->kh || p->W + 2 * p->pad < p->kw)
    return fail(SECN_EUNSUPPORTED, "unsupported shape: window larger than N or input");
  if (p->Hw && p->Ww) {  // explicit window; decim = 2 on input requests the polyphase packing
    if (derive_plan(n, p->Hw, p->Ww, p->decim == 2, p) != 0)
      return fail(SECN_EINVAL, "caller Hw,Ww (decim) invalid for this geometry");
    return SECN_OK;
  }
  // SECN_PLAN_BYTES (reading R6): minimise 8 L N (2GS + MG + 2MS) + 8 N MS; ties: fewer MGS, larger
  // Hw, larger Ww. SECN_PLAN_TIME (reading R6b): minimise the modelled device time of the
  // integer-issue-bound path, in ns per limb-poly of 4096 coefficients:
  //   13 per output limb-poly (INTT + mask), 1.3 per output limb-poly and input group (MAC),
  //   6 per input limb-poly (share add + NTT), and 0.3 x the bytes at 6.45 TB/s;
  // only plans with G <= 30 (above, the MAC's X^ tile and a 4-stage ring leave one CTA per SM
  // (ResNet-50 layer1 c3 takes 312 us at G = 32 and 241 us at G = 13;
  // tools/plan_sweep.py); G <= 32, the MAC kernel's limit, when no window has G <= 30;
  // ties: fewer bytes, larger Hw, larger Ww.
  for (uint32_t gmax = rule == SECN_PLAN_TIME ? 30u : 32u;; gmax = 32u) {
  secn_conv_plan_t best{};
  bool have = false;
  double best_t = 0;
  u128 best_cost = 0;
  uint64_t best_mgs = 0;
  const double limb_polys = 2.0 * n_limbs * (double)n / 4096.0;  // limb-polys of 4096 words per ct component
  const bool can_poly = p->stride > 1 && !(p->kh == 1 && p->kw == 1);
  for (int poly = 0; poly <= (rule == SECN_PLAN_TIME && can_poly ? 1 : 0); ++poly) {
    const uint32_t ps = poly ? p->stride : 1;
    const uint32_t khe = (p->kh + ps - 1) / ps, kwe = (p->kw + ps - 1) / ps;
    const uint32_t Hp = poly ? (p->H + 2 * p->pad + ps - 1) / ps
                              : ((p->kh == 1 && p->kw == 1 && p->stride > 1) ? (p->H + 2 * p->pad - 1) / p->stride + 1
                                                                             : p->H + 2 * p->pad);
    const uint32_t Wp = poly ? (p->W + 2 * p->pad + ps - 1) / ps
                              : ((p->kh == 1 && p->kw == 1 && p->stride > 1) ? (p->W + 2 * p->pad - 1) / p->stride + 1
                                                                             : p->W + 2 * p->pad);
    for (uint32_t Hw = khe; Hw <= Hp; ++Hw) {
      for (uint32_t Ww = kwe; Ww <= Wp; ++Ww) {
        if ((uint64_t)Hw * Ww > n) break;
        secn_conv_plan_t c = *p;
        if (derive_plan(n, Hw, Ww, poly, &c) != 0) continue;
        const u128 G = c.G, S = c.S, M = c.M;
        const u128 cost = (u128)8 * n_limbs * n * (2 * G * S + M * G + 2 * M * S) + (u128)8 * n * M * S;
        const uint64_t mgs = (uint64_t)(M * G * S);
        bool better;
        if (rule == SECN_PLAN_BYTES) {
          better = !have || cost < best_cost || (cost == best_cost && mgs < best_mgs) ||
                   (cost == best_cost && mgs == best_mgs && (Hw > best.Hw || (Hw == best.Hw && Ww > best.Ww)));
        } else {
          if (c.G > gmax) continue;
          const double ms = (double)(M * S), gs = (double)(G * S);
          const double t = 2.0 * limb_polys * (13.0 * ms + 1.3 * ms * (double)c.G + 6.0 * gs) + 0.3 * (double)cost / 6450.0;
          better = !have || t < best_t * (1 - 1e-12) ||
                   (t <= best_t * (1 + 1e-12) &&
                    (cost < best_cost || (cost == best_cost && (Hw > best.Hw || (Hw == best.Hw && Ww > best.Ww)))));
          if (better) best_t = t;
        }
        if (better) best = c, best_cost = cost, best_mgs = mgs, have = true;
      }
    }
  }
  if (!have && gmax < 32u) continue;  // no window with G <= 30: allow up to the kernel's limit
  if (!have) return fail(SECN_EUNSUPPORTED, "unsupported shape: no window fits N");
  *p = best;
  return SECN_OK;
  }
}

int secn_conv_plan(uint32_t log_n, uint32_t n_limbs /* coef_words64 */, secn_conv_plan_t* p) {
  return secn_conv_plan_ex(log_n, n_limbs, SECN_PLAN_TIME, p);
}

// ---- residue-buffer calls, generic over the context's word size ----
static int ntt_impl(secn_ctx* ctx, uint32_t bits, void* polys, size_t n_polys, void* stream, bool inverse) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (n_polys && !polys) return fail(SECN_EINVAL, "NULL polys");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const char* name = inverse ? "secn_ntt_inv" : "secn_ntt_fwd";
  if (int st = check_range(ctx, polys, n_polys * ctx->L * ctx->n, 0, s, name)) return st;
  cudaError_t e = inverse ? secn::launch_ntt_inv(ctx->dc, polys, n_polys * ctx->L, s)
                          : secn::launch_ntt_fwd(ctx->dc, polys, polys, n_polys * ctx->L, nullptr, s);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, name);
}

static int preprocess_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const uint64_t* kernel,
                           void* w_ntt, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  if (!kernel || !w_ntt) return fail(SECN_EINVAL, "NULL buffer");
  if (ctx->log_n > 14) return fail(SECN_EUNSUPPORTED, "convolutions need log_n <= 14 (N = 2^15 is NTT-only)");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t kw = (size_t)plan->M * plan->C * plan->kh * plan->kw;
  if (int st = check_range(ctx, kernel, kw, 1, s, "secn_preprocess_weights kernel")) return st;
  const secn::PlanDev pd = plan_dev(plan);
  cudaError_t e = secn::launch_pack_weights(ctx->dc, pd, kernel, w_ntt, s);
  if (e == cudaSuccess) e = secn::launch_ntt_fwd(ctx->dc, w_ntt, w_ntt, (size_t)plan->M * plan->G * ctx->L, nullptr, s);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_preprocess_weights");
}

static int enc_add_impl(secn_ctx* ctx, uint32_t bits, void* ct, const uint64_t* v, size_t n, void* stream,
                        const char* name) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (n && (!ct || !v)) return fail(SECN_EINVAL, "NULL buffer");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check_range(ctx, v, n * ctx->n, 1, s, name)) return st;
  cudaError_t e = secn::launch_enc_add(ctx->dc, ct, v, n, s);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, name);
}

int secn_ntt_fwd(secn_ctx* ctx, uint64_t* polys, size_t n_polys, void* stream) {
  SECN_NVTX();
  return ntt_impl(ctx, 64, polys, n_polys, stream, false);
}
int secn_ntt_inv(secn_ctx* ctx, uint64_t* polys, size_t n_polys, void* stream) {
  SECN_NVTX();
  return ntt_impl(ctx, 64, polys, n_polys, stream, true);
}
int secn32_ntt_fwd(secn_ctx* ctx, uint32_t* polys, size_t n_polys, void* stream) {
  SECN_NVTX();
  return ntt_impl(ctx, 32, polys, n_polys, stream, false);
}
int secn32_ntt_inv(secn_ctx* ctx, uint32_t* polys, size_t n_polys, void* stream) {
  SECN_NVTX();
  return ntt_impl(ctx, 32, polys, n_polys, stream, true);
}

int secn_preprocess_weights(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* kernel, uint64_t* w_ntt,
                            void* stream) {
  SECN_NVTX();
  return preprocess_impl(ctx, 64, plan, kernel, w_ntt, stream);
}
int secn32_preprocess_weights(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* kernel, uint32_t* w_ntt,
                              void* stream) {
  SECN_NVTX();
  return preprocess_impl(ctx, 32, plan, kernel, w_ntt, stream);
}

int secn_share_add(secn_ctx* ctx, uint64_t* ct, const uint64_t* x0, size_t n, void* stream) {
  SECN_NVTX();
  return enc_add_impl(ctx, 64, ct, x0, n, stream, "secn_share_add");
}
int secn_mask_add(secn_ctx* ctx, uint64_t* ct, const uint64_t* r, size_t n, void* stream) {
  SECN_NVTX();
  return enc_add_impl(ctx, 64, ct, r, n, stream, "secn_mask_add");
}
int secn32_share_add(secn_ctx* ctx, uint32_t* ct, const uint64_t* x0, size_t n, void* stream) {
  SECN_NVTX();
  return enc_add_impl(ctx, 32, ct, x0, n, stream, "secn32_share_add");
}
int secn32_mask_add(secn_ctx* ctx, uint32_t* ct, const uint64_t* r, size_t n, void* stream) {
  SECN_NVTX();
  return enc_add_impl(ctx, 32, ct, r, n, stream, "secn32_mask_add");
}

// Workspace of one layer call: the NTT-domain inputs X^ [G*S][2][L][N], then (full calls with a
// mask) the encoded mask em [M*S][L][N] (k_mask_encode), both in the context's word size.
static size_t xhat_bytes(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return (size_t)plan->G * plan->S * 2 * ctx->L * ctx->n * (ctx->word_bits / 8);
}
static size_t xhat_bytes_aligned(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return (xhat_bytes(ctx, plan) + 255) & ~(size_t)255;
}
static size_t em_bytes(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return (size_t)plan->M * plan->S * ctx->L * ctx->n * (ctx->word_bits / 8);
}

size_t secn_he_conv2d_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  if (!ctx || !plan) return 0;
  return xhat_bytes_aligned(ctx, plan) + em_bytes(ctx, plan);
}

// stage -1 = the whole layer; 0 / 1 / 2 = one launch group. `chained`: the caller launched this
// stage's predecessor stage itself just before (internal.h, "Pre-wait reads"); always true for -1.
// The mask (A7) arrives one of three ways: r (the tail loads and encodes it per limb, and writes
// y0); gen != NULL (full calls: drawn on the device, reading R17 -- k_mask_encode, launched right
// after the forward NTT, writes the encoded words em into the workspace and y0, and the tail adds
// em); or em_in != NULL (full calls: encoded beforehand by secn_mask_encode, the tail adds it).
// Stage calls (0, 1, 2) need only X^ in the workspace.
static int he_conv2d_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, int stage, const void* ct_in,
                          const uint64_t* x0, const void* w_ntt, const uint64_t* r, void* ct_out, uint64_t* y0,
                          void* workspace, size_t ws_bytes, void* stream, bool chained = false,
                          const secn::MaskGen* gen = nullptr, const void* em_in = nullptr) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  if (stage < -1 || stage > 2) return fail(SECN_EINVAL, "stage %d not in {0,1,2}", stage);
  if (!ct_in || !w_ntt || !ct_out || !workspace) return fail(SECN_EINVAL, "NULL buffer");
  if (ctx->log_n > 14) return fail(SECN_EUNSUPPORTED, "convolutions need log_n <= 14 (N = 2^15 is NTT-only)");
  if (y0 && !r && !gen) return fail(SECN_EINVAL, "y0 needs the mask r");
  const bool encode = stage == -1 && gen != nullptr;
  if (ws_bytes < (encode ? secn_he_conv2d_workspace(ctx, plan) : xhat_bytes(ctx, plan)))
    return fail(SECN_EINVAL, "workspace too small");
  if (((uintptr_t)workspace | (uintptr_t)ct_in | (uintptr_t)ct_out | (uintptr_t)w_ntt | (uintptr_t)r |
       (uintptr_t)em_in) & 15)
    return fail(SECN_EINVAL, "buffers must be 16-byte aligned");
  if (plan->G > 32u) return fail(SECN_EUNSUPPORTED, "G=%u input channel groups too many", plan->G);
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  // n_out: rows of r / ct_out; n_act: the output ciphertexts this call computes (its s-slice)
  const size_t n_in = (size_t)plan->G * plan->S, n_out = (size_t)plan->M * plan->S, N = ctx->n;
  const size_t n_act = (size_t)plan->M * (plan->s_count ? plan->s_count : plan->S);
  if (stage <= 0) {
    if (int st = check_range(ctx, ct_in, n_in * 2 * ctx->L * N, 0, s, "secn_he_conv2d ct_in")) return st;
    if (int st = check_range(ctx, x0, n_in * N, 1, s, "secn_he_conv2d x0")) return st;
  }
  if (stage == -1 || stage == 2)
    if (int st = check_range(ctx, r, n_out * N, 1, s, "secn_he_conv2d r")) return st;
  const secn::PlanDev pd = plan_dev(plan);
  cudaError_t e = cudaSuccess;
  if (stage == -1 || stage == 0) e = secn::launch_ntt_fwd(ctx->dc, ct_in, workspace, n_in * 2 * ctx->L, x0, s);  // A6+A1
  const void* em = em_in;
  if (e == cudaSuccess && encode) {  // A7 (+A8) drawn and encoded on the SMs the forward NTT leaves idle
    void* emw = static_cast<unsigned char*>(workspace) + xhat_bytes_aligned(ctx, plan);
    e = secn::launch_mask_encode(ctx->dc, pd, n_act, nullptr, *gen, emw, y0, s, true);
    em = emw;
  }
  // A4 + A2 levels 0..7
  const bool ch = chained || stage == -1;
  if (e == cudaSuccess && stage == -1 && secn::fused_applies(ctx->dc, pd)) {  // MAC + INTT + mask in one kernel
    e = secn::launch_layer_fused(ctx->dc, pd, workspace, w_ntt, ct_out, em ? nullptr : r, em ? nullptr : y0, s, true,
                                 const_cast<void*>(em));
    return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_he_conv2d");
  }
  if (e == cudaSuccess && (stage == -1 || stage == 1))
    e = secn::launch_mac(ctx->dc, pd, workspace, w_ntt, ct_out, s, ch);
  if (e == cudaSuccess && (stage == -1 || stage == 2))  // A2 (levels 8..) + A7 (+A8)
    e = secn::launch_ntt_inv_tail(ctx->dc, ct_out, n_act * 2 * ctx->L, em ? nullptr : r, em ? nullptr : y0, pd, s, ch,
                                  em);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_he_conv2d");
}

int secn_he_conv2d(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                   const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, void* workspace, size_t ws_bytes,
                   void* stream) {
  SECN_NVTX();
  return he_conv2d_impl(ctx, 64, plan, -1, ct_in, x0, w_ntt, r, ct_out, nullptr, workspace, ws_bytes, stream);
}

int secn_he_conv2d_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                      const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
                      size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_impl(ctx, 64, plan, -1, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}

int secn32_he_conv2d_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                        const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, uint64_t* y0, void* workspace,
                        size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_impl(ctx, 32, plan, -1, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}

// f4 ("online/offline/no NTT preprocessing"): the weights arrive in
// coefficient form and are packed + transformed inside the online call, into workspace scratch
// after X^; then the same three launches as secn_he_conv2d_ex.
static int check_gen(const secn_mask_gen_t* g, secn::MaskGen* out) {
  if (!g) return fail(SECN_EINVAL, "NULL mask generator");
  out->seed = g->seed, out->stream = g->stream, out->ct0 = g->ct0;
  return SECN_OK;
}

size_t secn_he_conv2d_gen_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return secn_he_conv2d_workspace(ctx, plan);  // the drawn mask goes straight into the encoded-mask buffer
}

static int he_conv2d_gen_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                              const uint64_t* x0, const void* w_ntt, const secn_mask_gen_t* gen, void* ct_out,
                              uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  secn::MaskGen g;
  if (int st = check_gen(gen, &g)) return st;
  return he_conv2d_impl(ctx, bits, plan, -1, ct_in, x0, w_ntt, nullptr, ct_out, y0, workspace, ws_bytes, stream, true,
                        &g);
}

int secn_he_conv2d_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                       const uint64_t* w_ntt, const secn_mask_gen_t* gen, uint64_t* ct_out, uint64_t* y0,
                       void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_gen_impl(ctx, 64, plan, ct_in, x0, w_ntt, gen, ct_out, y0, workspace, ws_bytes, stream);
}
int secn32_he_conv2d_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                         const uint32_t* w_ntt, const secn_mask_gen_t* gen, uint32_t* ct_out, uint64_t* y0,
                         void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_gen_impl(ctx, 32, plan, ct_in, x0, w_ntt, gen, ct_out, y0, workspace, ws_bytes, stream);
}

size_t secn_mask_encoded_bytes(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  if (!ctx || !plan) return 0;
  return em_bytes(ctx, plan);
}

int secn_mask_encode(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* r, const secn_mask_gen_t* gen,
                     void* em, uint64_t* y0, void* stream) {
  SECN_NVTX();
  if (int st = check_ctx(ctx)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  if (!em || (!r && !gen) || (r && gen)) return fail(SECN_EINVAL, "need em and exactly one of r, gen");
  if (((uintptr_t)em | (uintptr_t)r) & 15) return fail(SECN_EINVAL, "buffers must be 16-byte aligned");
  secn::MaskGen g{0, 0, 0};
  if (gen)
    if (int st = check_gen(gen, &g)) return st;
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check_range(ctx, r, (size_t)plan->M * plan->S * ctx->n, 1, s, "secn_mask_encode r")) return st;
  const secn::PlanDev pd = plan_dev(plan);
  cudaError_t e = secn::launch_mask_encode(ctx->dc, pd, (size_t)plan->M * pd.sn, r, g, em, y0, s, false);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_mask_encode");
}

static int he_conv2d_em_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                             const uint64_t* x0, const void* w_ntt, const void* em, void* ct_out, void* workspace,
                             size_t ws_bytes, void* stream) {
  if (!em) return fail(SECN_EINVAL, "NULL encoded mask");
  return he_conv2d_impl(ctx, bits, plan, -1, ct_in, x0, w_ntt, nullptr, ct_out, nullptr, workspace, ws_bytes, stream,
                        true, nullptr, em);
}
int secn_he_conv2d_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                      const uint64_t* w_ntt, const uint64_t* em, uint64_t* ct_out, void* workspace, size_t ws_bytes,
                      void* stream) {
  SECN_NVTX();
  return he_conv2d_em_impl(ctx, 64, plan, ct_in, x0, w_ntt, em, ct_out, workspace, ws_bytes, stream);
}
int secn32_he_conv2d_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                        const uint32_t* w_ntt, const uint32_t* em, uint32_t* ct_out, void* workspace, size_t ws_bytes,
                        void* stream) {
  SECN_NVTX();
  return he_conv2d_em_impl(ctx, 32, plan, ct_in, x0, w_ntt, em, ct_out, workspace, ws_bytes, stream);
}

int secn_mask_draw(secn_ctx* ctx, const secn_mask_gen_t* gen, size_t n_ct, uint64_t* r, void* stream) {
  SECN_NVTX();
  if (int st = check_ctx(ctx)) return st;
  secn::MaskGen g;
  if (int st = check_gen(gen, &g)) return st;
  if (n_ct && !r) return fail(SECN_EINVAL, "NULL buffer");
  if ((uintptr_t)r & 15) return fail(SECN_EINVAL, "r must be 16-byte aligned");
  DeviceGuard guard(ctx->device);
  cudaError_t e = secn::launch_mask_draw(ctx->dc, g, n_ct, r, (cudaStream_t)stream);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_mask_draw");
}

static size_t conv_ws_aligned(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return (secn_he_conv2d_workspace(ctx, plan) + 255) & ~(size_t)255;
}

size_t secn_he_conv2d_online_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  if (!ctx || !plan) return 0;
  return conv_ws_aligned(ctx, plan) + (size_t)plan->M * plan->G * ctx->L * ctx->n * (ctx->word_bits / 8);
}

static int he_conv2d_online_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                                 const uint64_t* x0, const uint64_t* kernel, const uint64_t* r, void* ct_out,
                                 uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  if (!workspace || !kernel) return fail(SECN_EINVAL, "NULL buffer");
  if (ws_bytes < secn_he_conv2d_online_workspace(ctx, plan)) return fail(SECN_EINVAL, "workspace too small");
  void* w_ntt = static_cast<unsigned char*>(workspace) + conv_ws_aligned(ctx, plan);
  if (int st = preprocess_impl(ctx, bits, plan, kernel, w_ntt, stream)) return st;
  return he_conv2d_impl(ctx, bits, plan, -1, ct_in, x0, w_ntt, r, ct_out, y0, workspace, conv_ws_aligned(ctx, plan),
                        stream);
}

int secn_he_conv2d_online(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                          const uint64_t* kernel, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
                          size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_online_impl(ctx, 64, plan, ct_in, x0, kernel, r, ct_out, y0, workspace, ws_bytes, stream);
}

int secn32_he_conv2d_online(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                            const uint64_t* kernel, const uint64_t* r, uint32_t* ct_out, uint64_t* y0,
                            void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_online_impl(ctx, 32, plan, ct_in, x0, kernel, r, ct_out, y0, workspace, ws_bytes, stream);
}

// ---- f3: fully connected (matrix-vector) layers ----

int secn_fc_plan(uint32_t log_n, uint32_t coef_words64, secn_fc_plan_t* p) {
  if (!p) return fail(SECN_EINVAL, "NULL plan");
  if (log_n < 1 || log_n > 20 || coef_words64 < 1) return fail(SECN_EUNSUPPORTED, "bad log_n / coef_words64");
  if (!p->n_i || !p->n_o) return fail(SECN_EINVAL, "empty matrix");
  const uint64_t n = 1ull << log_n, lim = p->n_i < n ? p->n_i : n;
  if (p->nib > lim) return fail(SECN_EINVAL, "nib=%u not in [1, min(n_i, N)]", p->nib);
  // reading R15: minimise 8 W N (2G + MG + 2M) + 8 N M; ties: fewer MG, then larger nib
  u128 best_cost = 0, best_mg = 0;
  uint32_t best = 0;
  for (uint64_t a = p->nib ? p->nib : 1; a <= (p->nib ? p->nib : lim); ++a) {
    const uint64_t b = p->n_o < n / a ? p->n_o : n / a;
    const uint64_t G = (p->n_i + a - 1) / a, M = (p->n_o + b - 1) / b;
    const u128 cost = (u128)8 * coef_words64 * n * (2 * G + M * G + 2 * M) + (u128)8 * n * M;
    const u128 mg = (u128)M * G;
    if (!best || cost < best_cost || (cost == best_cost && (mg < best_mg || (mg == best_mg && a > best)))) {
      best = (uint32_t)a, best_cost = cost, best_mg = mg;
    }
  }
  p->nib = best;
  p->nob = p->n_o < n / best ? p->n_o : (uint32_t)(n / best);
  p->G = (p->n_i + best - 1) / best;
  p->M = (p->n_o + p->nob - 1) / p->nob;
  return SECN_OK;
}

static int check_fc_plan(const secn_ctx* ctx, const secn_fc_plan_t* p) {
  if (!p) return fail(SECN_EINVAL, "NULL plan");
  secn_fc_plan_t q = *p;
  q.nob = q.G = q.M = 0;
  if (!p->nib || secn_fc_plan(ctx->log_n, 1, &q) != SECN_OK || q.nob != p->nob || q.G != p->G || q.M != p->M)
    return fail(SECN_EINVAL, "fc plan fields do not match secn_fc_plan() for this matrix and N");
  if (ctx->log_n > 14) return fail(SECN_EUNSUPPORTED, "fc layers need log_n <= 14 (N = 2^15 is NTT-only)");
  return SECN_OK;
}

static secn::PlanDev fc_plan_dev(const secn_fc_plan_t* p) {
  secn::PlanDev d{};
  d.kind = 1, d.M = p->M, d.G = p->G, d.S = 1, d.C = p->n_i, d.nib = p->nib, d.nob = p->nob, d.no = p->n_o;
  d.s0 = 0, d.sn = 1;
  return d;
}

static int fc_preprocess_impl(secn_ctx* ctx, uint32_t bits, const secn_fc_plan_t* plan, const uint64_t* W,
                              void* w_ntt, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_fc_plan(ctx, plan)) return st;
  if (!W || !w_ntt) return fail(SECN_EINVAL, "NULL buffer");
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check_range(ctx, W, (size_t)plan->n_o * plan->n_i, 1, s, "secn_fc_preprocess_weights W")) return st;
  const secn::PlanDev pd = fc_plan_dev(plan);
  cudaError_t e = secn::launch_pack_fc_weights(ctx->dc, pd, W, w_ntt, s);
  if (e == cudaSuccess) e = secn::launch_ntt_fwd(ctx->dc, w_ntt, w_ntt, (size_t)plan->M * plan->G * ctx->L, nullptr, s);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_fc_preprocess_weights");
}

size_t secn_he_fc_workspace(const secn_ctx* ctx, const secn_fc_plan_t* plan) {
  if (!ctx || !plan) return 0;
  return (size_t)plan->G * 2 * ctx->L * ctx->n * (ctx->word_bits / 8);
}

static int he_fc_impl(secn_ctx* ctx, uint32_t bits, const secn_fc_plan_t* plan, const void* ct_in, const uint64_t* x0,
                      const void* w_ntt, const uint64_t* r, void* ct_out, uint64_t* y0, void* workspace,
                      size_t ws_bytes, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_fc_plan(ctx, plan)) return st;
  if (!ct_in || !w_ntt || !ct_out || !workspace) return fail(SECN_EINVAL, "NULL buffer");
  if (y0 && !r) return fail(SECN_EINVAL, "y0 needs the mask r");
  if (ws_bytes < secn_he_fc_workspace(ctx, plan)) return fail(SECN_EINVAL, "workspace too small");
  if (((uintptr_t)workspace | (uintptr_t)ct_in | (uintptr_t)ct_out | (uintptr_t)w_ntt) & 15)
    return fail(SECN_EINVAL, "buffers must be 16-byte aligned");
  if (plan->G > 32u) return fail(SECN_EUNSUPPORTED, "G=%u input blocks too many", plan->G);
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t N = ctx->n;
  if (int st = check_range(ctx, ct_in, (size_t)plan->G * 2 * ctx->L * N, 0, s, "secn_he_fc ct_in")) return st;
  if (int st = check_range(ctx, x0, (size_t)plan->G * N, 1, s, "secn_he_fc x0")) return st;
  if (int st = check_range(ctx, r, (size_t)plan->M * N, 1, s, "secn_he_fc r")) return st;
  const secn::PlanDev pd = fc_plan_dev(plan);
  cudaError_t e = secn::launch_ntt_fwd(ctx->dc, ct_in, workspace, (size_t)plan->G * 2 * ctx->L, x0, s);
  if (e == cudaSuccess) e = secn::launch_mac(ctx->dc, pd, workspace, w_ntt, ct_out, s, true);
  if (e == cudaSuccess)
    e = secn::launch_ntt_inv_tail(ctx->dc, ct_out, (size_t)plan->M * 2 * ctx->L, r, y0, pd, s, true);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_he_fc");
}

int secn_fc_preprocess_weights(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* W, uint64_t* w_ntt,
                               void* stream) {
  SECN_NVTX();
  return fc_preprocess_impl(ctx, 64, plan, W, w_ntt, stream);
}
int secn32_fc_preprocess_weights(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* W, uint32_t* w_ntt,
                                 void* stream) {
  SECN_NVTX();
  return fc_preprocess_impl(ctx, 32, plan, W, w_ntt, stream);
}
int secn_he_fc(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
               const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0, void* workspace,
               size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_fc_impl(ctx, 64, plan, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}
int secn32_he_fc(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                 const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, uint64_t* y0, void* workspace,
                 size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_fc_impl(ctx, 32, plan, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}

// ---- f2: modulus switching + coefficient extraction of the outputs (reading R16) ----

static int make_ms(const secn_ctx* ctx, uint32_t keep, secn::MsConsts* ms) {
  const uint32_t L = ctx->L;
  if (ctx->log_n != 12) return fail(SECN_EUNSUPPORTED, "extracted outputs need N = 4096");
  if (keep < 1 || keep >= L) return fail(SECN_EUNSUPPORTED, "keep_limbs=%u not in [1, L-1] (L=%u)", keep, L);
  std::memset(ms, 0, sizeof *ms);
  ms->Lk = keep;
  u128 P = 1;
  for (uint32_t j = keep; j < L; ++j) P *= ctx->primes[j];
  if (P * (L - keep) >= ((u128)1 << 63)) return fail(SECN_EUNSUPPORTED, "dropped primes' product too large (> 2^62)");
  if (L - keep > (ctx->word_bits == 64 ? 1u : 2u))
    return fail(SECN_EUNSUPPORTED, "at most %u dropped limbs", ctx->word_bits == 64 ? 1u : 2u);
  ms->P = (uint64_t)P;
  auto comp = [&](uint64_t w, uint64_t q) {
    return ctx->word_bits == 64 ? shoup_companion(w, q) : (uint64_t)((((u128)w) << 32) / q);
  };
  for (uint32_t j = keep; j < L; ++j) {
    const uint64_t q = ctx->primes[j], pq = ms->P / q;
    ms->pq[j] = pq;
    ms->inv[j] = powmod(pq % q, q - 2, q);
    ms->inv_p[j] = comp(ms->inv[j], q);
  }
  for (uint32_t i = 0; i < keep; ++i) {
    const uint64_t q = ctx->primes[i];
    ms->pinv[i] = powmod(ms->P % q, q - 2, q);
    ms->pinv_p[i] = comp(ms->pinv[i], q);
  }
  return SECN_OK;
}

// X^ [G*S][2][L][N], Y^ [M*S][2][L][N] (the MAC's output, levels 0..7 applied), em [M*S][L][N]
size_t secn_he_conv2d_lwe_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  if (!ctx || !plan) return 0;
  const size_t wb = ctx->word_bits / 8;
  return xhat_bytes_aligned(ctx, plan) + (size_t)plan->M * plan->S * 2 * ctx->L * ctx->n * wb + em_bytes(ctx, plan);
}

static int he_conv2d_lwe_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                              const uint64_t* x0, const void* w_ntt, const uint64_t* r, uint32_t keep, void* a_out,
                              void* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream,
                              const secn::MaskGen* gen = nullptr, const void* em_in = nullptr) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  secn::MsConsts ms;
  if (int st = make_ms(ctx, keep, &ms)) return st;
  if (!ct_in || !w_ntt || !a_out || !b_out || !workspace) return fail(SECN_EINVAL, "NULL buffer");
  if (ws_bytes < secn_he_conv2d_lwe_workspace(ctx, plan)) return fail(SECN_EINVAL, "workspace too small");
  if (y0 && !r && !gen) return fail(SECN_EINVAL, "y0 needs the mask r");
  if (((uintptr_t)workspace | (uintptr_t)ct_in | (uintptr_t)w_ntt | (uintptr_t)r | (uintptr_t)em_in) & 15)
    return fail(SECN_EINVAL, "buffers must be 16-byte aligned");
  if (plan->G > 32u) return fail(SECN_EUNSUPPORTED, "G=%u input channel groups too many", plan->G);
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n_in = (size_t)plan->G * plan->S, n_out = (size_t)plan->M * plan->S, N = ctx->n;
  const secn::PlanDev pd = plan_dev(plan);
  const size_t n_act = (size_t)plan->M * pd.sn;
  if (int st = check_range(ctx, ct_in, n_in * 2 * ctx->L * N, 0, s, "secn_he_conv2d_lwe ct_in")) return st;
  if (int st = check_range(ctx, x0, n_in * N, 1, s, "secn_he_conv2d_lwe x0")) return st;
  if (int st = check_range(ctx, r, n_out * N, 1, s, "secn_he_conv2d_lwe r")) return st;
  // workspace: X^, then Y^ (levels 0..7 applied), then the encoded mask
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  void* yhat = ws + xhat_bytes_aligned(ctx, plan);
  // the mask: r (encoded in the tail), drawn (gen: encoded into the workspace right after the
  // forward NTT), or encoded beforehand (em_in)
  const void* em = em_in;
  void* emw = gen ? ws + xhat_bytes_aligned(ctx, plan) + n_out * 2 * ctx->L * N * (ctx->word_bits / 8) : nullptr;
  cudaError_t e = secn::launch_ntt_fwd(ctx->dc, ct_in, workspace, n_in * 2 * ctx->L, x0, s);  // A6 + A1
  if (e == cudaSuccess && gen) {
    e = secn::launch_mask_encode(ctx->dc, pd, n_act, nullptr, *gen, emw, y0, s, true);  // A7 (+A8)
    em = emw;
  }
  if (e == cudaSuccess) e = secn::launch_mac(ctx->dc, pd, workspace, w_ntt, yhat, s, true);  // A4 + INTT 0..7
  if (e == cudaSuccess)  // INTT 8.. + mask + modulus switch + extraction
    e = secn::launch_ntt_inv_tail_lwe(ctx->dc, ms, yhat, n_act, em ? nullptr : r, a_out, b_out, em ? nullptr : y0, pd,
                                      s, true, em);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_he_conv2d_lwe");
}

size_t secn_he_conv2d_lwe_gen_workspace(const secn_ctx* ctx, const secn_conv_plan_t* plan) {
  return secn_he_conv2d_lwe_workspace(ctx, plan);  // the drawn mask goes straight into the encoded-mask buffer
}

static int he_conv2d_lwe_gen_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                                  const uint64_t* x0, const void* w_ntt, const secn_mask_gen_t* gen, uint32_t keep,
                                  void* a_out, void* b_out, uint64_t* y0, void* workspace, size_t ws_bytes,
                                  void* stream) {
  secn::MaskGen g;
  if (int st = check_gen(gen, &g)) return st;
  return he_conv2d_lwe_impl(ctx, bits, plan, ct_in, x0, w_ntt, nullptr, keep, a_out, b_out, y0, workspace, ws_bytes,
                            stream, &g);
}

static int he_conv2d_lwe_em_impl(secn_ctx* ctx, uint32_t bits, const secn_conv_plan_t* plan, const void* ct_in,
                                 const uint64_t* x0, const void* w_ntt, const void* em, uint32_t keep, void* a_out,
                                 void* b_out, void* workspace, size_t ws_bytes, void* stream) {
  if (!em) return fail(SECN_EINVAL, "NULL encoded mask");
  return he_conv2d_lwe_impl(ctx, bits, plan, ct_in, x0, w_ntt, nullptr, keep, a_out, b_out, nullptr, workspace,
                            ws_bytes, stream, nullptr, em);
}
int secn_he_conv2d_lwe_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                          const uint64_t* w_ntt, const uint64_t* em, uint32_t keep_limbs, uint64_t* a_out,
                          uint64_t* b_out, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_em_impl(ctx, 64, plan, ct_in, x0, w_ntt, em, keep_limbs, a_out, b_out, workspace, ws_bytes,
                               stream);
}
int secn32_he_conv2d_lwe_em(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                            const uint32_t* w_ntt, const uint32_t* em, uint32_t keep_limbs, uint32_t* a_out,
                            uint32_t* b_out, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_em_impl(ctx, 32, plan, ct_in, x0, w_ntt, em, keep_limbs, a_out, b_out, workspace, ws_bytes,
                               stream);
}

int secn_he_conv2d_lwe_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                           const uint64_t* w_ntt, const secn_mask_gen_t* gen, uint32_t keep_limbs, uint64_t* a_out,
                           uint64_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_gen_impl(ctx, 64, plan, ct_in, x0, w_ntt, gen, keep_limbs, a_out, b_out, y0, workspace,
                                ws_bytes, stream);
}
int secn32_he_conv2d_lwe_gen(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                             const uint32_t* w_ntt, const secn_mask_gen_t* gen, uint32_t keep_limbs, uint32_t* a_out,
                             uint32_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_gen_impl(ctx, 32, plan, ct_in, x0, w_ntt, gen, keep_limbs, a_out, b_out, y0, workspace,
                                ws_bytes, stream);
}

int secn_he_conv2d_lwe(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                       const uint64_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint64_t* a_out,
                       uint64_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_impl(ctx, 64, plan, ct_in, x0, w_ntt, r, keep_limbs, a_out, b_out, y0, workspace, ws_bytes,
                            stream);
}
int secn32_he_conv2d_lwe(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                         const uint32_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint32_t* a_out,
                         uint32_t* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_conv2d_lwe_impl(ctx, 32, plan, ct_in, x0, w_ntt, r, keep_limbs, a_out, b_out, y0, workspace, ws_bytes,
                            stream);
}

size_t secn_he_fc_lwe_workspace(const secn_ctx* ctx, const secn_fc_plan_t* plan) {
  if (!ctx || !plan) return 0;
  const size_t wb = ctx->word_bits / 8;
  return ((secn_he_fc_workspace(ctx, plan) + 255) & ~(size_t)255) + (size_t)plan->M * 2 * ctx->L * ctx->n * wb;
}

static int he_fc_lwe_impl(secn_ctx* ctx, uint32_t bits, const secn_fc_plan_t* plan, const void* ct_in,
                          const uint64_t* x0, const void* w_ntt, const uint64_t* r, uint32_t keep, void* a_out,
                          void* b_out, uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  if (int st = check_ctx(ctx, bits)) return st;
  if (int st = check_fc_plan(ctx, plan)) return st;
  secn::MsConsts ms;
  if (int st = make_ms(ctx, keep, &ms)) return st;
  if (!ct_in || !w_ntt || !a_out || !b_out || !workspace) return fail(SECN_EINVAL, "NULL buffer");
  if (ws_bytes < secn_he_fc_lwe_workspace(ctx, plan)) return fail(SECN_EINVAL, "workspace too small");
  if (y0 && !r) return fail(SECN_EINVAL, "y0 needs the mask r");
  if (((uintptr_t)workspace | (uintptr_t)ct_in | (uintptr_t)w_ntt) & 15)
    return fail(SECN_EINVAL, "buffers must be 16-byte aligned");
  if (plan->G > 32u) return fail(SECN_EUNSUPPORTED, "G=%u input blocks too many", plan->G);
  DeviceGuard guard(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t xb = (secn_he_fc_workspace(ctx, plan) + 255) & ~(size_t)255;
  void* yhat = static_cast<unsigned char*>(workspace) + xb;
  const secn::PlanDev pd = fc_plan_dev(plan);
  if (int st = check_range(ctx, ct_in, (size_t)plan->G * 2 * ctx->L * ctx->n, 0, s, "secn_he_fc_lwe ct_in")) return st;
  if (int st = check_range(ctx, x0, (size_t)plan->G * ctx->n, 1, s, "secn_he_fc_lwe x0")) return st;
  if (int st = check_range(ctx, r, (size_t)plan->M * ctx->n, 1, s, "secn_he_fc_lwe r")) return st;
  cudaError_t e = secn::launch_ntt_fwd(ctx->dc, ct_in, workspace, (size_t)plan->G * 2 * ctx->L, x0, s);
  if (e == cudaSuccess) e = secn::launch_mac(ctx->dc, pd, workspace, w_ntt, yhat, s, true);
  if (e == cudaSuccess) e = secn::launch_ntt_inv_tail_lwe(ctx->dc, ms, yhat, plan->M, r, a_out, b_out, y0, pd, s, true);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_he_fc_lwe");
}

int secn_he_fc_lwe(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint64_t* ct_in, const uint64_t* x0,
                   const uint64_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint64_t* a_out, uint64_t* b_out,
                   uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_fc_lwe_impl(ctx, 64, plan, ct_in, x0, w_ntt, r, keep_limbs, a_out, b_out, y0, workspace, ws_bytes, stream);
}
int secn32_he_fc_lwe(secn_ctx* ctx, const secn_fc_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                     const uint32_t* w_ntt, const uint64_t* r, uint32_t keep_limbs, uint32_t* a_out, uint32_t* b_out,
                     uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  return he_fc_lwe_impl(ctx, 32, plan, ct_in, x0, w_ntt, r, keep_limbs, a_out, b_out, y0, workspace, ws_bytes, stream);
}

int secn_he_conv2d_stage(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint64_t* ct_in,
                         const uint64_t* x0, const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out,
                         void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  if (stage < 0 || stage > 2) return fail(SECN_EINVAL, "stage %d not in {0,1,2}", stage);
  return he_conv2d_impl(ctx, 64, plan, stage, ct_in, x0, w_ntt, r, ct_out, nullptr, workspace, ws_bytes, stream);
}

int secn32_he_conv2d(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint32_t* ct_in, const uint64_t* x0,
                     const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out, void* workspace, size_t ws_bytes,
                     void* stream) {
  SECN_NVTX();
  return he_conv2d_impl(ctx, 32, plan, -1, ct_in, x0, w_ntt, r, ct_out, nullptr, workspace, ws_bytes, stream);
}

int secn32_he_conv2d_stage(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint32_t* ct_in,
                           const uint64_t* x0, const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out,
                           void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  if (stage < 0 || stage > 2) return fail(SECN_EINVAL, "stage %d not in {0,1,2}", stage);
  return he_conv2d_impl(ctx, 32, plan, stage, ct_in, x0, w_ntt, r, ct_out, nullptr, workspace, ws_bytes, stream);
}

int secn_he_conv2d_stage_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint64_t* ct_in,
                            const uint64_t* x0, const uint64_t* w_ntt, const uint64_t* r, uint64_t* ct_out, uint64_t* y0,
                            void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  if (stage < 0 || stage > 2) return fail(SECN_EINVAL, "stage %d not in {0,1,2}", stage);
  return he_conv2d_impl(ctx, 64, plan, stage, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}

int secn32_he_conv2d_stage_ex(secn_ctx* ctx, const secn_conv_plan_t* plan, int stage, const uint32_t* ct_in,
                              const uint64_t* x0, const uint32_t* w_ntt, const uint64_t* r, uint32_t* ct_out,
                              uint64_t* y0, void* workspace, size_t ws_bytes, void* stream) {
  SECN_NVTX();
  if (stage < 0 || stage > 2) return fail(SECN_EINVAL, "stage %d not in {0,1,2}", stage);
  return he_conv2d_impl(ctx, 32, plan, stage, ct_in, x0, w_ntt, r, ct_out, y0, workspace, ws_bytes, stream);
}

int secn_extract_share(secn_ctx* ctx, const secn_conv_plan_t* plan, const uint64_t* r, uint64_t* y0, void* stream) {
  SECN_NVTX();
  if (int st = check_ctx(ctx)) return st;
  if (int st = check_plan(ctx, plan)) return st;
  if (!r || !y0) return fail(SECN_EINVAL, "NULL buffer");
  DeviceGuard guard(ctx->device);
  cudaError_t e = secn::launch_extract_share(ctx->dc, plan_dev(plan), r, y0, (cudaStream_t)stream);
  return e == cudaSuccess ? SECN_OK : cuda_fail(e, "secn_extract_share");
}

}  // extern "C"
