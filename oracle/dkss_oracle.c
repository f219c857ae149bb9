/*
 * dkss_oracle.c -- CPU ORACLE for the DKSS hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is a plain-C restatement of the reference's pure-Python DKSS
 * multiplication (/root/reference/pkg/src/bigmul/dkss.py).  It exists so that
 * tests/ can check the CUDA path bit-for-bit and so that bench.py can time a
 * CPU baseline ("cpu_baseline.kind": "port").  Only tests/, the smoke() in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
 * load it; the product path (paper_1503_04955_b200) never does.
 *
 * Pinning: tests/test_oracle_golden.py checks every function below against
 * vectors the reference itself produced (tools/make_golden.py ->
 * tests/golden/*.npz), so the oracle's parity is anchored on the reference.
 *
 * Function map (reference file:line it follows):
 *   modp_*            poly_add/poly_sub/poly_neg       dkss.py:26-43
 *   xpow              poly_mul_xpow                    dkss.py:46-61
 *   oracle_rmul       r_mul (+ _ks_mul)                dkss.py:401-431
 *                     (the Kronecker-packed integer product computes the acyclic
 *                      convolution z_k = sum_{i+j=k} x_i y_j exactly; we form the
 *                      same z_k directly and apply out[k] = (z_k - z_{m+k}) mod p,
 *                      dkss.py:417-420)
 *   fft_eval_alpha    fft_eval with PolyAlphaRing      fft.py:70-109, dkss.py:64-91
 *   shuffle           shuffle / shuffle_indices        fft.py:15-44
 *   oracle_fft        dkss_fft                         dkss.py:443-495
 *   oracle_encode     dkss_encode (+ bit_slices)       dkss.py:381-398, words.py:307-329
 *   oracle_decode     dkss_decode (+ join_bits)        dkss.py:498-513, words.py:332-349
 *   oracle_dmul       dmul body                        dkss.py:536-548
 *
 * Layout shared with the GPU path: a polynomial is uint32[2M][m][L]
 * (L = ceil(d/32) little-endian limbs per canonical residue).
 *
 * Threads: OpenMP over the independent column / row / pointwise loops and over
 * batch pairs (the reference itself is single-threaded).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define MAXL 8              /* max u32 limbs per residue (d <= 256) */
#define MAXW (2 * MAXL + 2) /* accumulator digits */

typedef struct {
  int N, M, m, u, L, mu;
  uint32_t p[MAXL];
  uint32_t inv2M[MAXL];
  uint32_t* rho;     /* mu * m * L, canonical rho^s */
  /* Knuth-D normalisation of p */
  int shift;
  uint32_t pn[MAXL]; /* p << shift */
  long long ks_calls;
} oplan;

/* ------------------------------------------------------------------------ */
/* multiprecision helpers on little-endian u32 digit arrays                  */

static int cmp_n(const uint32_t* a, const uint32_t* b, int n) {
  for (int i = n - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  return 0;
}

static int is_zero(const uint32_t* a, int n) {
  for (int i = 0; i < n; ++i)
    if (a[i]) return 0;
  return 1;
}

/* r = (a + b) mod p  -- poly_add, dkss.py:26-31 */
static void add_mod(uint32_t* r, const uint32_t* a, const uint32_t* b, const oplan* P) {
  uint32_t s[MAXL + 1];
  uint64_t c = 0;
  for (int i = 0; i < P->L; ++i) { c += (uint64_t)a[i] + b[i]; s[i] = (uint32_t)c; c >>= 32; }
  s[P->L] = (uint32_t)c;
  uint32_t pp[MAXL + 1];
  memcpy(pp, P->p, 4 * P->L); pp[P->L] = 0;
  if (cmp_n(s, pp, P->L + 1) >= 0) {
    int64_t br = 0;
    for (int i = 0; i <= P->L; ++i) { int64_t t = (int64_t)s[i] - pp[i] - br; s[i] = (uint32_t)t; br = t < 0; }
  }
  memcpy(r, s, 4 * P->L);
}

/* r = (a - b) mod p  -- poly_sub, dkss.py:34-39 */
static void sub_mod(uint32_t* r, const uint32_t* a, const uint32_t* b, const oplan* P) {
  uint32_t d[MAXL];
  int64_t br = 0;
  for (int i = 0; i < P->L; ++i) { int64_t t = (int64_t)a[i] - b[i] - br; d[i] = (uint32_t)t; br = t < 0; }
  if (br) {
    uint64_t c = 0;
    for (int i = 0; i < P->L; ++i) { c += (uint64_t)d[i] + P->p[i]; d[i] = (uint32_t)c; c >>= 32; }
  }
  memcpy(r, d, 4 * P->L);
}

/* r = -a mod p  (p - c if c else 0) -- poly_neg, dkss.py:42-43 */
static void neg_mod(uint32_t* r, const uint32_t* a, const oplan* P) {
  if (is_zero(a, P->L)) { memset(r, 0, 4 * P->L); return; }
  int64_t br = 0;
  for (int i = 0; i < P->L; ++i) { int64_t t = (int64_t)P->p[i] - a[i] - br; r[i] = (uint32_t)t; br = t < 0; }
}

/* rem = x mod p for an n-digit x (Knuth algorithm D, remainder only) */
static void mod_p(uint32_t* rem, const uint32_t* x, int n, const oplan* P) {
  int L = P->L;
  int lp = L;
  while (lp > 1 && P->pn[lp - 1] == 0) --lp; /* cannot happen for normalised p, kept for safety */
  uint32_t u[MAXW + 2];
  /* u = x << shift, one extra digit */
  if (P->shift) {
    u[n] = x[n - 1] >> (32 - P->shift);
    for (int i = n - 1; i > 0; --i) u[i] = (x[i] << P->shift) | (x[i - 1] >> (32 - P->shift));
    u[0] = x[0] << P->shift;
  } else {
    memcpy(u, x, 4 * n);
    u[n] = 0;
  }
  const uint32_t* v = P->pn;
  uint64_t vtop = v[lp - 1], vsec = lp > 1 ? v[lp - 2] : 0;
  for (int j = n - lp; j >= 0; --j) {
    uint64_t num = ((uint64_t)u[j + lp] << 32) | u[j + lp - 1];
    uint64_t qhat = num / vtop, rhat = num % vtop;
    while (qhat >> 32 || (lp > 1 && qhat * vsec > ((rhat << 32) | u[j + lp - 2]))) {
      --qhat;
      rhat += vtop;
      if (rhat >> 32) break;
    }
    /* u[j .. j+lp] -= qhat * v */
    int64_t br = 0;
    uint64_t carry = 0;
    for (int i = 0; i < lp; ++i) {
      uint64_t prod = qhat * v[i] + carry;
      carry = prod >> 32;
      int64_t t = (int64_t)u[i + j] - (int64_t)(uint32_t)prod - br;
      u[i + j] = (uint32_t)t;
      br = t < 0;
    }
    int64_t t = (int64_t)u[j + lp] - (int64_t)carry - br;
    u[j + lp] = (uint32_t)t;
    if (t < 0) { /* add back */
      uint64_t c = 0;
      for (int i = 0; i < lp; ++i) { c += (uint64_t)u[i + j] + v[i]; u[i + j] = (uint32_t)c; c >>= 32; }
      u[j + lp] += (uint32_t)c;
    }
  }
  /* remainder = u[0..lp) >> shift */
  for (int i = 0; i < L; ++i) {
    uint32_t lo = i < lp ? u[i] : 0, hi = i + 1 < lp ? u[i + 1] : 0;
    rem[i] = P->shift ? (lo >> P->shift) | (hi << (32 - P->shift)) : lo;
  }
}

/* acc (W digits) += a * b (L x L digits) */
static void mac(uint32_t* acc, int W, const uint32_t* a, const uint32_t* b, int L) {
  for (int i = 0; i < L; ++i) {
    uint64_t c = 0;
    uint64_t ai = a[i];
    if (!ai) continue;
    for (int j = 0; j < L; ++j) {
      c += ai * b[j] + acc[i + j];
      acc[i + j] = (uint32_t)c;
      c >>= 32;
    }
    for (int k = i + L; c && k < W; ++k) { c += acc[k]; acc[k] = (uint32_t)c; c >>= 32; }
  }
}

/* r = a * b mod p */
static void mul_mod(uint32_t* r, const uint32_t* a, const uint32_t* b, const oplan* P) {
  uint32_t t[MAXW];
  memset(t, 0, sizeof t);
  mac(t, 2 * P->L, a, b, P->L);
  mod_p(r, t, 2 * P->L, P);
}

/* ------------------------------------------------------------------------ */
/* ring R = P[alpha]/(alpha^m+1); an element is m consecutive residues      */

#define RES(v, i, k, P) ((v) + ((size_t)(i) * (P)->m + (k)) * (P)->L)

/* out = x * alpha^e  -- poly_mul_xpow, dkss.py:46-61 (out must not alias x) */
static void xpow(uint32_t* out, const uint32_t* x, int e, const oplan* P) {
  int m = P->m, L = P->L;
  e %= 2 * m;
  if (e < 0) e += 2 * m;
  for (int i = 0; i < m; ++i) {
    int j = i + e, neg = 0;
    while (j >= m) { j -= m; neg ^= 1; }
    if (neg) neg_mod(out + (size_t)j * L, x + (size_t)i * L, P);
    else memcpy(out + (size_t)j * L, x + (size_t)i * L, 4 * L);
  }
}

/* out = x * y in R  -- r_mul, dkss.py:401-420 */
static void rmul_elem(uint32_t* out, const uint32_t* x, const uint32_t* y, oplan* P) {
  int m = P->m, L = P->L, W = 2 * L + 2;
  uint32_t z[2 * 64][MAXW];
  for (int k = 0; k < 2 * m; ++k) memset(z[k], 0, 4 * W);
  for (int i = 0; i < m; ++i) {
    const uint32_t* xi = x + (size_t)i * L;
    if (is_zero(xi, L)) continue;
    for (int j = 0; j < m; ++j) mac(z[i + j], W, xi, y + (size_t)j * L, L);
  }
  for (int k = 0; k < m; ++k) {
    uint32_t lo[MAXL], hi[MAXL];
    mod_p(lo, z[k], W, P);
    mod_p(hi, z[m + k], W, P);
    sub_mod(out + (size_t)k * L, lo, hi, P);
  }
#pragma omp atomic
  P->ks_calls++;
}

/* in-place radix-2 DIT on a pre-shuffled vector of n ring elements with root
 * alpha^(2m/n) -- fft_eval + PolyAlphaRing, fft.py:70-109 / dkss.py:64-91 */
static void fft_eval_alpha(uint32_t* v, int n, oplan* P) {
  int m = P->m, L = P->L;
  size_t es = (size_t)m * L;
  int scale = 2 * m / n;
  uint32_t* t = malloc(4 * es);
  uint32_t* u = malloc(4 * es);
  for (int size = 2; size <= n; size <<= 1) {
    int half = size >> 1, step = n / size;
    for (int base = 0; base < n; base += size)
      for (int k = 0; k < half; ++k) {
        uint32_t* a = v + (size_t)(base + k) * es;
        uint32_t* b = v + (size_t)(base + half + k) * es;
        if (k == 0) memcpy(t, b, 4 * es);
        else xpow(t, b, k * step * scale, P);
        memcpy(u, a, 4 * es);
        for (int c = 0; c < m; ++c) {
          sub_mod(b + (size_t)c * L, u + (size_t)c * L, t + (size_t)c * L, P);
          add_mod(a + (size_t)c * L, u + (size_t)c * L, t + (size_t)c * L, P);
        }
      }
  }
  free(t);
  free(u);
}

static int bitrev(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

static int ilog2(long long n) {
  int k = 0;
  while ((1LL << k) < n) ++k;
  return k;
}

/* dkss_fft, dkss.py:443-495: v[i] <- a(rho^i), natural order in and out */
static void fft_rec(uint32_t* v, long long length, long long base_pow, oplan* P) {
  int m = P->m, L = P->L;
  size_t es = (size_t)m * L;
  int two_m = 2 * m;
  if (length <= two_m) { /* shuffle + inner DFT, dkss.py:458-463 */
    int bits = ilog2(length);
    uint32_t* tmp = malloc(4 * es * length);
    for (int j = 0; j < length; ++j) memcpy(tmp + j * es, v + (size_t)bitrev(j, bits) * es, 4 * es);
    fft_eval_alpha(tmp, (int)length, P);
    memcpy(v, tmp, 4 * es * length);
    free(tmp);
    return;
  }
  long long mu = length / two_m;
  int bits = ilog2(two_m);
  uint32_t* abar = malloc(4 * es * length); /* abar[vv][l] */
  /* inner DFTs, dkss.py:473-478 */
#pragma omp parallel for schedule(static) if (mu >= 8)
  for (long long l = 0; l < mu; ++l) {
    uint32_t* el = malloc(4 * es * two_m);
    for (int j = 0; j < two_m; ++j) memcpy(el + j * es, v + ((size_t)bitrev(j, bits) * mu + l) * es, 4 * es);
    fft_eval_alpha(el, two_m, P);
    for (int vv = 0; vv < two_m; ++vv) memcpy(abar + ((size_t)vv * mu + l) * es, el + vv * es, 4 * es);
    free(el);
  }
  /* twiddles + outer DFTs, dkss.py:480-495 */
  long long top_mu = mu * base_pow, mask = top_mu - 1;
  int sh = ilog2(top_mu);
#pragma omp parallel for schedule(dynamic, 1)
  for (int vv = 0; vv < two_m; ++vv) {
    uint32_t* row = abar + (size_t)vv * mu * es;
    uint32_t* tw = malloc(4 * es);
    uint32_t* tmp = malloc(4 * es);
    if (vv) {
      long long e = 0, step = vv * base_pow;
      for (long long l = 1; l < mu; ++l) {
        e += step;
        const uint32_t* rs = P->rho + (size_t)(e & mask) * es;
        xpow(tw, rs, (int)((e >> sh) % (2 * m)), P);
        rmul_elem(tmp, row + l * es, tw, P);
        memcpy(row + l * es, tmp, 4 * es);
      }
    }
    fft_rec(row, mu, base_pow * two_m, P);
    for (long long f = 0; f < mu; ++f) memcpy(v + ((size_t)f * two_m + vv) * es, row + f * es, 4 * es);
    free(tw);
    free(tmp);
  }
  free(abar);
}

/* ------------------------------------------------------------------------ */
/* exported API                                                              */

void* oracle_plan_create(int N, int M, int m, int u, int L, const uint32_t* p, const uint32_t* rho_powers,
                         const uint32_t* inv2M) {
  if (L < 1 || L > MAXL || m > 64) return NULL;
  oplan* P = calloc(1, sizeof(oplan));
  P->N = N; P->M = M; P->m = m; P->u = u; P->L = L; P->mu = M / m;
  memcpy(P->p, p, 4 * L);
  memcpy(P->inv2M, inv2M, 4 * L);
  size_t n = (size_t)P->mu * m * L;
  P->rho = malloc(4 * n);
  memcpy(P->rho, rho_powers, 4 * n);
  int top = L - 1;
  while (top > 0 && p[top] == 0) --top;
  P->shift = __builtin_clz(p[top]);
  /* pn = p << shift, within L digits (top digit has room by construction) */
  for (int i = L - 1; i >= 0; --i) {
    uint32_t lo = i > 0 ? p[i - 1] : 0;
    P->pn[i] = P->shift ? (p[i] << P->shift) | (lo >> (32 - P->shift)) : p[i];
  }
  if (top != L - 1) { free(P->rho); free(P); return NULL; } /* d must exceed 32(L-1) */
  return P;
}

void oracle_plan_destroy(void* h) {
  oplan* P = h;
  if (!P) return;
  free(P->rho);
  free(P);
}

long long oracle_ks_calls(void* h, int reset) {
  oplan* P = h;
  long long v = P->ks_calls;
  if (reset) P->ks_calls = 0;
  return v;
}

void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int oracle_max_threads(void) { return omp_get_max_threads(); }

/* x, y, out: count ring elements each; out = x * y elementwise */
void oracle_rmul(void* h, const uint32_t* x, const uint32_t* y, uint32_t* out, long long count) {
  oplan* P = h;
  size_t es = (size_t)P->m * P->L;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < count; ++i) rmul_elem(out + i * es, x + i * es, y + i * es, P);
}

/* bits [u*idx, u*idx+u) of the operand a (na limbs) */
static void get_slot(uint32_t* dst, const uint32_t* a, long long na, long long bit, int u, int L) {
  memset(dst, 0, 4 * L);
  for (int b = 0; b < u; ++b) {
    long long pos = bit + b, li = pos >> 5;
    if (li >= na) break;
    if ((a[li] >> (pos & 31)) & 1u) dst[b >> 5] |= 1u << (b & 31);
  }
}

/* dkss_encode, dkss.py:381-398 -> poly uint32[2M][m][L] */
int oracle_encode(void* h, const uint32_t* a, long long na, uint32_t* poly) {
  oplan* P = h;
  int m = P->m, L = P->L, half = m / 2;
  /* a < 2^N required, dkss.py:389-390 */
  for (long long i = 0; i < na; ++i) {
    long long lo = 32 * i;
    if (!a[i]) continue;
    int top = 31 - __builtin_clz(a[i]);
    if (lo + top >= P->N) return -1;
  }
  memset(poly, 0, 4 * (size_t)2 * P->M * m * L);
#pragma omp parallel for schedule(static)
  for (long long b = 0; b < P->M; ++b)
    for (int i = 0; i < half; ++i)
      get_slot(RES(poly, b, i, P), a, na, (long long)P->u * (b * half + i), P->u, L);
  return 0;
}

void oracle_fft(void* h, uint32_t* poly) {
  oplan* P = h;
  fft_rec(poly, 2LL * P->M, 1, P);
}

/* dkss_decode, dkss.py:498-513: out = sum_l sum_k (v[-l mod 2M][k] / 2M) * 2^(u(l m/2 + k)) */
void oracle_decode(void* h, const uint32_t* v, uint32_t* out, long long nout) {
  oplan* P = h;
  int m = P->m, L = P->L, half = m / 2;
  long long two_M = 2LL * P->M;
  memset(out, 0, 4 * nout);
  uint32_t c[MAXL];
  for (long long l = 0; l < two_M; ++l) {
    long long src = (two_M - l) % two_M;
    for (int k = 0; k < m; ++k) {
      mul_mod(c, RES(v, src, k, P), P->inv2M, P);
      long long bit = (long long)P->u * (l * half + k);
      long long li = bit >> 5;
      int sh = bit & 31;
      /* add c << sh at limb li, propagate carry */
      uint64_t carry = 0;
      for (int j = 0; j <= L; ++j) {
        uint64_t part = j < L ? ((uint64_t)c[j] << sh) : 0;
        uint64_t prev = j > 0 ? (sh ? (uint64_t)c[j - 1] >> (32 - sh) : 0) : 0;
        uint64_t word = (uint32_t)part | (uint32_t)prev;
        if (li + j >= nout) { if (word || carry) { /* overflow beyond product length */ } break; }
        carry += (uint64_t)out[li + j] + word;
        out[li + j] = (uint32_t)carry;
        carry >>= 32;
      }
      for (long long t = li + L + 1; carry && t < nout; ++t) {
        carry += out[t];
        out[t] = (uint32_t)carry;
        carry >>= 32;
      }
    }
  }
}

/* pointwise products of two transformed polynomials (dkss.py:544-545) */
void oracle_pointwise(void* h, const uint32_t* a, const uint32_t* b, uint32_t* out) {
  oplan* P = h;
  oracle_rmul(h, a, b, out, 2LL * P->M);
}

/* full product for operands below 2^N (dkss.py:536-548); returns 0 or <0 */
int oracle_dmul(void* h, const uint32_t* a, long long na, const uint32_t* b, long long nb, uint32_t* out,
                long long nout) {
  oplan* P = h;
  size_t n = (size_t)2 * P->M * P->m * P->L;
  uint32_t* ap = malloc(4 * n);
  uint32_t* bp = malloc(4 * n);
  int rc = oracle_encode(h, a, na, ap);
  if (!rc) rc = oracle_encode(h, b, nb, bp);
  if (!rc) {
    oracle_fft(h, ap);
    oracle_fft(h, bp);
    oracle_rmul(h, ap, bp, ap, 2LL * P->M);
    oracle_fft(h, ap);
    oracle_decode(h, ap, out, nout);
  }
  free(ap);
  free(bp);
  return rc;
}

/* independent products, one pair per thread (the batched config) */
int oracle_dmul_batch(void* h, int batch, const uint32_t* a, const uint32_t* b, long long nlimbs, uint32_t* out,
                      long long nout) {
  int bad = 0;
  int outer = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(outer) reduction(| : bad)
  for (int i = 0; i < batch; ++i) {
    omp_set_num_threads(1);
    bad |= oracle_dmul(h, a + (size_t)i * nlimbs, nlimbs, b + (size_t)i * nlimbs, nlimbs, out + (size_t)i * nout,
                       nout) != 0;
  }
  return bad ? -1 : 0;
}
