// smul_capi.cuh -- host side of the SMUL multiply (include/smul.h); included at the end of
// dkss_capi.cu so it shares the launch helper, the error channel and the carry-scan kernels.
#pragma once
#include <algorithm>
#include "../../include/smul.h"
#include "smul_kernels.cuh"

struct smul_plan {
  int device = 0;
  long long N = 0, s = 0, n = 0;
  int m = 0, K = 0, KW = 0, Q = 1, omega_exp = 0;
  long long prod_limbs = 0;
  int nlv_max = 1;  // most DIT levels one FFT pass runs in shared memory
  size_t smem_pw = 0;  // pointwise kernel, warp-per-product form
  cudaStream_t stream = nullptr;
  int cap = 0;  // operands the workspace holds (a's and b's)
  long long cap_nc = 0;
  uint32_t *d_x = nullptr, *d_xt = nullptr, *d_o = nullptr, *d_ot = nullptr;
  uint32_t *d_ops = nullptr, *d_prod = nullptr, *d_gmask = nullptr, *d_pmask = nullptr, *d_bstat = nullptr;
  uint32_t* h_pin = nullptr;    // pinned staging of the digits entry point
  uint32_t* d_stage = nullptr;
  size_t pin_words = 0;
  std::mutex mu;
};

namespace {

constexpr int kSmulPwWarps = 4;
#ifndef DKSS_SMUL_WPP  // warps per product of the CTA-wide pointwise kernel (experiment override)
#define DKSS_SMUL_WPP 4  // measured: 4 beats 8 by 1.4-2.7% from 2^22 up, equal at 2^20
#endif
constexpr size_t kSmulFftSmemMax = 96 * 1024;

template <int Q>
int smul_set_attrs(smul_plan* P) {
  CUCHK(cudaFuncSetAttribute(k_smul_fft<Q, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmulFftSmemMax));
  CUCHK(cudaFuncSetAttribute(k_smul_fft<Q, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmulFftSmemMax));
  // the attribute is per kernel, not per plan: allow the largest plan this Q serves
  const int pw_max = kSmulPwWarps * (10 * 32 * Q + 8) * 4;
  CUCHK(cudaFuncSetAttribute(k_smul_pointwise<Q, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, pw_max));
  CUCHK(cudaFuncSetAttribute(k_smul_pointwise<Q, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, pw_max));
  CUCHK(cudaFuncSetAttribute(k_smul_pointwise<Q, DKSS_SMUL_WPP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (10 * 32 * Q + 8) * 4));
  CUCHK(cudaFuncSetAttribute(k_smul_pointwise<Q, DKSS_SMUL_WPP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (10 * 32 * Q + 8) * 4));
  return 0;
}

int smul_attrs(smul_plan* P) {
  switch (P->Q) {
    case 1: return smul_set_attrs<1>(P);
    case 2: return smul_set_attrs<2>(P);
    case 3: return smul_set_attrs<3>(P);
    case 6: return smul_set_attrs<6>(P);
    case 4: return smul_set_attrs<4>(P);
    case 8: return smul_set_attrs<8>(P);
    case 16: return smul_set_attrs<16>(P);
    case 32: return smul_set_attrs<32>(P);
  }
  return fail(DKSS_EINVAL, "unsupported limb count per lane %d", P->Q);
}

template <int Q>
void smul_fft_q(smul_plan* P, uint32_t* x, uint32_t* top, int npoly, bool inverse, bool normalise, cudaStream_t s,
                const SmulFftArgs* enc) {
  SmulFftArgs A{};
  if (enc) {  // encode fused into the first pass
    A.enc_a = enc->enc_a;
    A.enc_b = enc->enc_b;
    A.enc_na = enc->enc_na;
    A.enc_s = enc->enc_s;
    A.enc_batch = enc->enc_batch;
  }
  A.x = x;
  A.top = top;
  A.log_n = P->m;
  A.KW = P->KW;
  A.K = P->K;
  A.omega_fwd = P->omega_exp;
  A.inverse = inverse ? 1 : 0;
  // levels per pass: at most what shared memory and one warp per butterfly (<= 32 warps)
  // allow, fewer while the launch has under 96 CTAs (measured with the shorter passes first:
  // 2^20 65 us at 96, 68 at 64, 67 at 148; fewer, deeper passes beat covering all 148 SMs);
  // then split the levels evenly
  static const long long min_ctas = [] {
    const char* e = DKSS_KNOB("DKSS_SMUL_MINCTA");  // experiment knob
    return e ? atoll(e) : 96LL;
  }();
  int nlv = P->nlv_max;
  while (nlv > 3 && (P->n >> nlv) * npoly < min_ctas) --nlv;
  const int npass = (P->m + nlv - 1) / nlv;
  for (int i = 0, lv = 0; i < npass; ++i) {
    // the shorter passes first (2^18 -7%, 2^20 -6%): the first forward pass also builds its
    // elements from the operand limbs
    const int nl = (P->m - lv) / (npass - i);
    A.lv0 = lv;
    A.nlv = nl;
    lv += nl;
    A.post_e = (normalise && i + 1 == npass) ? (2 * P->K - P->m) % (2 * P->K) : -1;
    const int G = 1 << A.nlv;
    const size_t smem = (size_t)G * smul_elem_stride(P->KW, smul_pad<Q>()) * 4 + (size_t)G * 4;
    const int nt = std::max(32, G / 2 * 32);
    if (P->KW == 32 * Q)  // every limb slot live: the kernel drops its bounds checks
      launch_k(k_smul_fft<Q, true>, dim3((unsigned)(P->n >> A.nlv), npoly), dim3(nt), smem, s, A);
    else
      launch_k(k_smul_fft<Q, false>, dim3((unsigned)(P->n >> A.nlv), npoly), dim3(nt), smem, s, A);
    A.enc_a = nullptr;
  }
}

void smul_fft(smul_plan* P, uint32_t* x, uint32_t* top, int npoly, bool inverse, bool normalise, cudaStream_t s,
              const SmulFftArgs* enc = nullptr) {
  switch (P->Q) {
    case 1: return smul_fft_q<1>(P, x, top, npoly, inverse, normalise, s, enc);
    case 2: return smul_fft_q<2>(P, x, top, npoly, inverse, normalise, s, enc);
    case 3: return smul_fft_q<3>(P, x, top, npoly, inverse, normalise, s, enc);
    case 6: return smul_fft_q<6>(P, x, top, npoly, inverse, normalise, s, enc);
    case 4: return smul_fft_q<4>(P, x, top, npoly, inverse, normalise, s, enc);
    case 8: return smul_fft_q<8>(P, x, top, npoly, inverse, normalise, s, enc);
    case 16: return smul_fft_q<16>(P, x, top, npoly, inverse, normalise, s, enc);
    case 32: return smul_fft_q<32>(P, x, top, npoly, inverse, normalise, s, enc);
  }
}

// small K: a warp per product (4 per CTA); K >= 2080 (3+ limbs per lane): DKSS_SMUL_WPP warps per product
template <int Q>
void smul_pw_q(smul_plan* P, const SmulPwArgs& A, cudaStream_t s) {
  const bool full = P->KW == 32 * Q;
  if (Q >= 3) {
    constexpr int W = DKSS_SMUL_WPP;
    const dim3 g((unsigned)std::min<long long>(A.count, 148LL * 64 / W));
    const size_t sm = (size_t)(10 * P->KW + 8) * 4;
    if (full)
      launch_k(k_smul_pointwise<Q, W, true>, g, dim3(32 * W), sm, s, A);
    else
      launch_k(k_smul_pointwise<Q, W, false>, g, dim3(32 * W), sm, s, A);
    return;
  }
  const long long blocks = (A.count + kSmulPwWarps - 1) / kSmulPwWarps;
  const dim3 g((unsigned)std::min<long long>(blocks, 148LL * 16));
  if (full)
    launch_k(k_smul_pointwise<Q, 1, true>, g, dim3(32 * kSmulPwWarps), P->smem_pw, s, A);
  else
    launch_k(k_smul_pointwise<Q, 1, false>, g, dim3(32 * kSmulPwWarps), P->smem_pw, s, A);
}

void smul_pointwise(smul_plan* P, const SmulPwArgs& A, cudaStream_t s) {
  switch (P->Q) {
    case 1: return smul_pw_q<1>(P, A, s);
    case 2: return smul_pw_q<2>(P, A, s);
    case 3: return smul_pw_q<3>(P, A, s);
    case 6: return smul_pw_q<6>(P, A, s);
    case 4: return smul_pw_q<4>(P, A, s);
    case 8: return smul_pw_q<8>(P, A, s);
    case 16: return smul_pw_q<16>(P, A, s);
    case 32: return smul_pw_q<32>(P, A, s);
  }
}

void smul_free(smul_plan* P) {
  for (uint32_t** p : {&P->d_x, &P->d_xt, &P->d_o, &P->d_ot, &P->d_ops, &P->d_prod, &P->d_gmask, &P->d_pmask,
                       &P->d_bstat}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  P->cap = 0;
  P->cap_nc = 0;
}

// workspace for `ops` transforms (a's and b's) and products of nc limbs
int smul_ensure(smul_plan* P, int ops, long long nc) {
  if (ops <= P->cap && nc <= P->cap_nc) return 0;
  ops = std::max(ops, P->cap);
  nc = std::max(nc, P->cap_nc);
  smul_free(P);
  const size_t vec = (size_t)P->n * P->KW;
  const int prods = ops;  // products never outnumber the transforms
  const long long blocks = (nc + kDecThreads - 1) / kDecThreads;
  CUCHK(cudaMalloc(&P->d_x, (size_t)ops * vec * 4));
  CUCHK(cudaMalloc(&P->d_xt, (size_t)ops * P->n * 4));
  CUCHK(cudaMalloc(&P->d_o, (size_t)prods * vec * 4));
  CUCHK(cudaMalloc(&P->d_ot, (size_t)prods * P->n * 4));
  CUCHK(cudaMalloc(&P->d_ops, (size_t)ops * P->prod_limbs * 4));
  CUCHK(cudaMalloc(&P->d_prod, (size_t)prods * nc * 4));
  CUCHK(cudaMalloc(&P->d_gmask, (size_t)prods * blocks * kDecWarps * 4));
  CUCHK(cudaMalloc(&P->d_pmask, (size_t)prods * blocks * kDecWarps * 4));
  CUCHK(cudaMalloc(&P->d_bstat, (size_t)prods * blocks * 4));
  P->cap = ops;
  P->cap_nc = nc;
  return 0;
}

// the whole multiply, stream-ordered: encode, forward FFTs, pointwise, inverse FFT (+2^-m),
// overlap-add with carry resolution (bigmul/smul.py:238-249, 256-271)
int run_smul(smul_plan* P, int batch, const uint32_t* a, const uint32_t* b, long long na, uint32_t* c, long long nc,
             cudaStream_t s) {
  const bool sq = b == nullptr;
  const int ops = (sq ? 1 : 2) * batch;
  int rc;
  if ((rc = smul_ensure(P, ops, nc))) return rc;
  const long long vec = P->n * P->KW;
  SmulFftArgs enc{};  // encode (bit_slices + shuffle) fused into the first forward pass
  enc.enc_a = a;
  enc.enc_b = sq ? a : b;
  enc.enc_na = na;
  enc.enc_s = P->s;
  enc.enc_batch = batch;
  smul_fft(P, P->d_x, P->d_xt, ops, false, false, s, &enc);
  SmulPwArgs W{};
  W.x = P->d_x;
  W.xtop = P->d_xt;
  W.y = sq ? P->d_x : P->d_x + (size_t)batch * vec;
  W.ytop = sq ? P->d_xt : P->d_xt + (size_t)batch * P->n;
  W.out = P->d_o;
  W.otop = P->d_ot;
  W.log_n = P->m;
  W.KW = P->KW;
  W.count = (long long)batch * P->n;
  smul_pointwise(P, W, s);
  smul_fft(P, P->d_o, P->d_ot, batch, true, true, s);
  DecodeArgs A{};
  A.out = c;
  A.nout = nc;
  A.gmask = P->d_gmask;
  A.pmask = P->d_pmask;
  A.bstat = P->d_bstat;
  A.blocks_per_poly = (int)((nc + kDecThreads - 1) / kDecThreads);
  SmulDecodeArgs D{};
  D.x = P->d_o;
  D.log_n = P->m;
  D.KW = P->KW;
  D.s = P->s;
  D.s_log = (P->s & (P->s - 1)) ? -1 : ilog2i(P->s);
  launch_k(k_smul_decode1, dim3(A.blocks_per_poly * batch), dim3(kDecThreads), 0, s, A, D);
  launch_carry_tail(A, batch, s);
  CUCHK(cudaGetLastError());
  return 0;
}

long long bitlen_limbs(const uint32_t* a, size_t na) {
  while (na > 0 && a[na - 1] == 0) --na;
  return na ? (long long)(na - 1) * 32 + (32 - __builtin_clz(a[na - 1])) : 0;
}

}  // namespace

extern "C" {

int smul_plan_create(const smul_plan_desc* d, int device, smul_plan** out) {
  if (!d || !out) return fail(DKSS_EINVAL, "bad argument");
  *out = nullptr;
  if (d->m < 1 || d->m > 26) return fail(DKSS_EINVAL, "FFT depth m=%d outside [1, 26]", d->m);
  const long long n = 1LL << d->m;
  if (d->s < 1 || d->s * n != d->N) return fail(DKSS_EINVAL, "N must equal s * 2^m");  // bigmul/smul.py:37-38
  if (d->K % 32) return fail(DKSS_EINVAL, "K=%d not a multiple of 32 (device limbs)", d->K);
  if ((long long)d->K < d->m + 2 * d->s + 1) return fail(DKSS_EINVAL, "K below the convolution bound m + 2s + 1");
  if ((2LL * d->K) % n) return fail(DKSS_EINVAL, "outermost level needs n | 2K");  // bigmul/smul.py:43-45
  if ((long long)d->omega_exp * n != 2LL * d->K) return fail(DKSS_EINVAL, "omega_exp must be 2K/n");
  if (d->K > 32 * 1024) return fail(DKSS_EINVAL, "K=%d above the device limit 32768", d->K);
  auto* P = new smul_plan();
  P->device = device;
  P->N = d->N;
  P->m = d->m;
  P->n = n;
  P->s = d->s;
  P->K = d->K;
  P->KW = d->K / 32;
  P->omega_exp = d->omega_exp;
  P->prod_limbs = (d->N + 31) / 32;
  int q = (P->KW + 31) / 32, Q = 1;
  static const int kQs[] = {1, 2, 3, 4, 6, 8, 16, 32};  // limbs per lane the kernels are built for
  for (int qq : kQs)
    if (qq >= q) {
      Q = qq;
      break;
    }
  P->Q = Q;
  // FFT passes: up to 64 elements (32 butterfly warps) per CTA, as shared memory allows
  int nlv_max = 1;
  const size_t es = (size_t)P->KW + (P->KW + 31) / 32 + 1;  // padded element + its top word, upper bound
  while (nlv_max < 6 && nlv_max < d->m && (es * 4) << (nlv_max + 1) <= kSmulFftSmemMax) ++nlv_max;
  P->nlv_max = std::min(nlv_max, d->m);
  P->smem_pw = (size_t)kSmulPwWarps * (10 * P->KW + 8) * 4;
  int rc;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete P;
    return fail(DKSS_ECUDA, "smul_plan_create: %s", cudaGetErrorString(e));
  }
  if ((rc = smul_attrs(P))) {
    cudaStreamDestroy(P->stream);
    delete P;
    return rc;
  }
  *out = P;
  return DKSS_OK;
}

void smul_plan_destroy(smul_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  smul_free(P);
  if (P->h_pin) cudaFreeHost(P->h_pin);
  if (P->d_stage) cudaFree(P->d_stage);
  if (P->stream) cudaStreamDestroy(P->stream);
  delete P;
}

int64_t smul_product_limbs(const smul_plan* P) { return P ? P->prod_limbs : -1; }

int smul_mul_device(smul_plan* P, int batch, const uint32_t* a_dev, const uint32_t* b_dev, size_t n_limbs,
                    uint32_t* c_dev, size_t nc, void* stream) {
  if (!P || batch < 1 || !a_dev || !c_dev) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nc < P->prod_limbs) return fail(DKSS_EINVAL, "nc=%zu below the plan's %lld product limbs", nc, P->prod_limbs);
  // the fused encode reads N bits per operand: wider operands would lose their top slices
  if ((long long)n_limbs * 32 > P->N) return fail(DKSS_ERANGE, "operands of %zu limbs exceed the plan's N=%lld bits", n_limbs, P->N);
  if (2LL * batch > 65535) return fail(DKSS_EINVAL, "batch %d too large (grid y limit)", batch);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  return run_smul(P, batch, a_dev, b_dev, (long long)n_limbs, c_dev, (long long)nc, (cudaStream_t)stream);
}

int smul_mul(smul_plan* P, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint32_t* c, size_t nc) {
  if (!P || (!a && na) || (!b && nb) || (!c && nc)) return fail(DKSS_EINVAL, "bad argument");
  const long long ba = bitlen_limbs(a, na), bb = bitlen_limbs(b, nb);
  if (ba + bb > P->N) return fail(DKSS_ERANGE, "product of %lld + %lld bits exceeds N=%lld", ba, bb, P->N);
  const bool sq = a == b && na == nb;
  const size_t la = (size_t)(ba + 31) / 32, lb = (size_t)(bb + 31) / 32;
  const size_t nl = std::max<size_t>(1, std::max(la, lb));
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = smul_ensure(P, 2, P->prod_limbs))) return rc;
  cudaStream_t s = P->stream;
  if (nl > (size_t)P->prod_limbs) return fail(DKSS_ERANGE, "operand does not fit the plan");
  uint32_t* da = P->d_ops;
  uint32_t* db = P->d_ops + nl;
  CUCHK(cudaMemsetAsync(P->d_ops, 0, 2 * nl * 4, s));
  if (la) CUCHK(cudaMemcpyAsync(da, a, la * 4, cudaMemcpyHostToDevice, s));
  if (!sq && lb) CUCHK(cudaMemcpyAsync(db, b, lb * 4, cudaMemcpyHostToDevice, s));
  if ((rc = run_smul(P, 1, da, sq ? nullptr : db, (long long)nl, P->d_prod, P->prod_limbs, s))) return rc;
  std::vector<uint32_t> full((size_t)P->prod_limbs);
  CUCHK(cudaMemcpyAsync(full.data(), P->d_prod, full.size() * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  const size_t ncopy = std::min<size_t>(nc, full.size());
  for (size_t k = ncopy; k < full.size(); ++k)
    if (full[k]) return fail(DKSS_ERANGE, "product does not fit nc=%zu limbs", nc);
  if (ncopy) memcpy(c, full.data(), ncopy * 4);
  if (nc > ncopy) memset(c + ncopy, 0, (nc - ncopy) * 4);
  return DKSS_OK;
}

int smul_mul_digits(smul_plan* P, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int digit_bits,
                    uint32_t* c, size_t nc) {
  if (!P || (!a && na) || (!b && nb) || (!c && nc)) return fail(DKSS_EINVAL, "bad argument");
  const bool trusted = digit_bits & DKSS_DIGITS_TRUSTED;
  digit_bits &= ~DKSS_DIGITS_TRUSTED;
  if (digit_bits < 8 || digit_bits > 32) return fail(DKSS_EINVAL, "digit_bits=%d outside [8, 32]", digit_bits);
  const bool sq = a == b && na == nb;
  const uint32_t* ops[2] = {a, b};
  size_t nd[2] = {na, nb};
  long long bits[2];
  for (int q = 0; q < 2; ++q) {
    while (nd[q] > 0 && ops[q][nd[q] - 1] == 0) --nd[q];
    if (digit_bits < 32 && !trusted) {
      uint32_t any = 0;
      for (size_t i = 0; i < nd[q]; ++i) any |= ops[q][i];
      if (any >> digit_bits) return fail(DKSS_EINVAL, "a digit exceeds %d bits", digit_bits);
    }
    const uint32_t top = nd[q] ? ops[q][nd[q] - 1] : 0u;
    if (digit_bits < 32 && (top >> digit_bits)) return fail(DKSS_EINVAL, "a digit exceeds %d bits", digit_bits);
    bits[q] = nd[q] ? (long long)(nd[q] - 1) * digit_bits + (32 - __builtin_clz(top)) : 0;
  }
  if (bits[0] + bits[1] > P->N) return fail(DKSS_ERANGE, "product of %lld + %lld bits exceeds N=%lld", bits[0], bits[1], P->N);
  const size_t nl = (size_t)std::max<long long>(1, (std::max(bits[0], bits[1]) + 31) / 32);
  const int nops = sq ? 1 : 2;
  const size_t head = 2 * (size_t)(nops + 1);  // long long offsets, in u32 words
  const size_t cap = head + nd[0] + (sq ? 0 : nd[1]);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = smul_ensure(P, 2, P->prod_limbs))) return rc;
  const size_t pin_need = std::max(cap, (size_t)P->prod_limbs);
  if (pin_need > P->pin_words) {
    if (P->h_pin) cudaFreeHost(P->h_pin);
    if (P->d_stage) cudaFree(P->d_stage);
    P->h_pin = nullptr;
    P->d_stage = nullptr;
    P->pin_words = 0;
    CUCHK(cudaMallocHost(&P->h_pin, pin_need * 4));
    CUCHK(cudaMalloc(&P->d_stage, pin_need * 4));
    P->pin_words = pin_need;
  }
  long long* off = reinterpret_cast<long long*>(P->h_pin);
  off[0] = 0;
  off[1] = (long long)nd[0];
  if (!sq) off[2] = (long long)(nd[0] + nd[1]);
  if (nd[0]) memcpy(P->h_pin + head, a, nd[0] * 4);
  if (!sq && nd[1]) memcpy(P->h_pin + head + nd[0], b, nd[1] * 4);
  cudaStream_t s = P->stream;
  CUCHK(cudaMemcpyAsync(P->d_stage, P->h_pin, cap * 4, cudaMemcpyHostToDevice, s));
  RepackArgs R{};  // radix change on the device (k_repack_bits, shared with the DKSS entry point)
  R.stage = P->d_stage + head;
  R.off = reinterpret_cast<const long long*>(P->d_stage);
  R.dst = P->d_ops;
  R.ndst = (long long)nl;
  R.sbits = digit_bits;
  const int gx = (int)std::max<size_t>(1, std::min<size_t>((nl + 255) / 256, 592));
  launch_k(k_repack_bits, dim3(gx, nops), dim3(256), 0, s, R);
  if ((rc = run_smul(P, 1, P->d_ops, sq ? nullptr : P->d_ops + nl, (long long)nl, P->d_prod, P->prod_limbs, s)))
    return rc;
  CUCHK(cudaMemcpyAsync(P->h_pin, P->d_prod, P->prod_limbs * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  const size_t ncopy = std::min<size_t>(nc, (size_t)P->prod_limbs);
  for (size_t k = ncopy; k < (size_t)P->prod_limbs; ++k)
    if (P->h_pin[k]) return fail(DKSS_ERANGE, "product does not fit nc=%zu limbs", nc);
  if (ncopy) memcpy(c, P->h_pin, ncopy * 4);
  if (nc > ncopy) memset(c + ncopy, 0, (nc - ncopy) * 4);
  return DKSS_OK;
}

int smul_fft_host(smul_plan* P, uint32_t* x, uint32_t* top, int inverse) {
  if (!P || !x || !top) return fail(DKSS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = smul_ensure(P, 1, P->prod_limbs))) return rc;
  cudaStream_t s = P->stream;
  const size_t vec = (size_t)P->n * P->KW;
  for (long long i = 0; i < P->n; ++i)
    if (top[i] > 1 || (top[i] && std::any_of(x + i * P->KW, x + (i + 1) * P->KW, [](uint32_t w) { return w != 0; })))
      return fail(DKSS_EINVAL, "element %lld is not canonical in [0, 2^K]", i);
  CUCHK(cudaMemcpyAsync(P->d_x, x, vec * 4, cudaMemcpyHostToDevice, s));
  CUCHK(cudaMemcpyAsync(P->d_xt, top, P->n * 4, cudaMemcpyHostToDevice, s));
  smul_fft(P, P->d_x, P->d_xt, 1, inverse != 0, false, s);
  CUCHK(cudaGetLastError());
  CUCHK(cudaMemcpyAsync(x, P->d_x, vec * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaMemcpyAsync(top, P->d_xt, P->n * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  return DKSS_OK;
}

}  // extern "C"
