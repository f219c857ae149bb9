/*
 * smul.h -- C ABI of the Schoenhage-Strassen (SMUL) multiply in libdkss (sm_100a).
 *
 * SMUL is the reference's comparison baseline for DKSS: the thesis's
 * central measurement is T_DMUL / T_SMUL.  The reference implements it in Python
 * (bigmul/smul.py, bigmul/fermat.py) and registers it as ALGORITHMS["smul"]
 * (bigmul/dispatch.py:16); it has no FFI of its own.  This library implements the outermost,
 * cyclic level of smul (bigmul/smul.py:286-300 -> _smul_mod_int :219-249 ->
 * _cyclic_coeff_product :256-271): slices of s bits, a length-n = 2^m FFT over Z/(2^K+1)
 * with root 2^omega_exp, the pointwise products in Z/(2^K+1), the inverse FFT with the 2^-m
 * normalisation, and the overlap-add at stride s.  Pointwise products are computed directly
 * on the GPU instead of by recursive smul / Toom-3 (bigmul/smul.py:206-216): the same residues.
 *
 * Conventions as include/dkss.h: 0 / negative DKSS_E* status, dkss_last_error() for the
 * message; little-endian uint32 limbs; a plan handle is used by one host thread at a time.
 * The plan (N, m, s, K, omega_exp) is chosen by the host planner (smul_select_params,
 * bigmul/smul.py:128-153, restated in paper_1503_04955_b200/smul.py).
 */
#ifndef SMUL_H
#define SMUL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct smul_plan smul_plan;

/* field-for-field the outermost SmulPlan (bigmul/smul.py:20-30): N = s * 2^m, K a multiple of
 * 32 with K >= m + 2s + 1 and n | 2K, omega_exp = 2K / n, theta_exp = 0. */
typedef struct {
  int64_t N;
  int32_t m;
  int64_t s;
  int32_t K;
  int32_t omega_exp;
} smul_plan_desc;

int smul_plan_create(const smul_plan_desc* desc, int device, smul_plan** out);
void smul_plan_destroy(smul_plan* plan);

/* limbs of one product: ceil(N/32) */
int64_t smul_product_limbs(const smul_plan* plan);

/* c = a * b (replaces smul(a, b), bigmul/smul.py:286-300).  Host limbs; a*b must be < 2^N
 * (bit lengths summing to at most N, DKSS_ERANGE otherwise).  c gets nc limbs (zero padded;
 * DKSS_ERANGE if the product needs more).  a == b (same pointer and size) squares. */
int smul_mul(smul_plan* plan, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint32_t* c, size_t nc);

/* the same product from radix-2^digit_bits digit strings (8 <= digit_bits <= 32, one digit per
 * uint32, little endian; | DKSS_DIGITS_TRUSTED skips the digit range scan), e.g. CPython's
 * 30-bit int digits: staged to the device and repacked there (as dkss_mul_digits). */
int smul_mul_digits(smul_plan* plan, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int digit_bits,
                    uint32_t* c, size_t nc);

/* batch device multiply: a_dev, b_dev are [batch][n_limbs] (b_dev NULL squares a), c_dev is
 * [batch][nc] with nc >= smul_product_limbs.  Stream-ordered; products must be < 2^N. */
int smul_mul_device(smul_plan* plan, int batch, const uint32_t* a_dev, const uint32_t* b_dev, size_t n_limbs,
                    uint32_t* c_dev, size_t nc, void* stream);

/* stage parity: fft_eval (bigmul/fft.py:70-109) over the plan's FermatRing (bigmul/fermat.py:
 * 67-93) in place on host data: x is [n][K/32] limbs, top[n] the bit K of each canonical
 * element; input in shuffled (bit-reversed) order, output natural.  inverse != 0 uses
 * omega^-1 (FermatRing.inverse_ring). */
int smul_fft_host(smul_plan* plan, uint32_t* x, uint32_t* top, int inverse);

#ifdef __cplusplus
}
#endif

#endif /* SMUL_H */
