/*
 * dkss.h -- C ABI of libdkss (B200 / sm_100a DKSS large-integer multiplication).
 *
 * This is the drop-in boundary for the reference's DKSS multiply path.  The reference
 * (bigmul, pure Python) has no FFI of its own; its plugin surface is the ALGORITHMS
 * table entry  ALGORITHMS["dmul"] = lambda a, b, table, arena: dmul(a, b, table, arena)
 * (bigmul/dispatch.py:17) and the stage functions of bigmul/dkss.py.  Each entry point
 * below names the reference function it replaces; INTEGRATION.md shows the ctypes
 * binding a bigmul maintainer would add.
 *
 * Conventions
 *  - plain pointers and sizes; integers are little-endian uint32 limb arrays;
 *    polynomials are uint32[2M][m][L] (L = ceil(d/32) limbs per canonical residue).
 *  - every call returns 0 on success and a negative DKSS_E* code on failure;
 *    dkss_last_error() returns a thread-local message for the last failure.
 *  - the plan is built by the host planner (Python, bigmul/dkss.py:314-361 restated in
 *    paper_1503_04955_b200/plan.py); the library only uploads it (rho table -> Montgomery
 *    form) and owns device workspace.
 *  - a plan handle may be used by one host thread at a time; calls are synchronous for
 *    host pointers and stream-ordered for the *_device entry points.
 */
#ifndef DKSS_H
#define DKSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DKSS_OK 0
#define DKSS_EINVAL (-1)  /* bad argument / plan shape (reference: ValueError) */
#define DKSS_ECUDA (-2)   /* CUDA runtime failure */
#define DKSS_ERANGE (-3)  /* operand does not fit the plan (bigmul/dkss.py:389-390) */
#define DKSS_ENOMEM (-4)

typedef struct dkss_plan dkss_plan;

/* Plan description, field-for-field the reference DkssPlan (bigmul/dkss.py:97-146)
 * restricted to what the device needs. */
typedef struct {
  int64_t N;                   /* inputs < 2^N */
  int32_t M, m, u;             /* outer length M (transform 2M), inner length m, bits per piece */
  int32_t L;                   /* u32 limbs per residue, ceil(d/32) */
  const uint32_t* p;           /* L limbs, the Proth prime p (z = 1) */
  const uint32_t* rho_powers;  /* (M/m) * m * L limbs: rho^s, s < M/m (DkssPlan.rho_powers) */
} dkss_plan_desc;

typedef struct {
  int64_t N;
  int32_t M, m, u, L;
  int32_t levels;           /* radix-2m column passes per transform */
  int32_t base_len;         /* length of the base-case DFT */
  int64_t poly_bytes;       /* one polynomial, 2M*m*L*4 */
  int64_t operand_limbs;    /* ceil(N/32) */
  int64_t product_limbs;    /* ceil(2N/32) */
  int64_t ring_products;    /* r_mul-equivalents per multiply: 3*twiddles + 2M (== ks_calls) */
  int64_t twiddles_per_fft; /* (2m-1)(mu-1) summed over levels (bigmul/dkss.py:483-492) */
  int32_t launches_per_mul; /* kernels launched by one dkss_mul_device call */
  int64_t workspace_bytes;  /* device workspace currently held */
  int64_t footprint_bytes;  /* device bytes one multiply of host operands holds: twiddle tables, two
                               polynomials, operand staging, operands, product, decode scratch
                               (the arena figure dmul reports, cf. bigmul/dkss.py:538-539) */
} dkss_plan_info;

/* Kernel-shape choices of a plan.  Zero-initialised options (or dkss_plan_create) pick the
 * measured-fastest shape for the plan; the others exist for parity tests of every variant. */
#define DKSS_ROWS_AUTO 0        /* per plan */
#define DKSS_ROWS_LAUNCHES 1    /* row phase as three ticketed persistent launches */
#define DKSS_ROWS_PERSISTENT 2  /* row phase as one dependency-driven kernel (k_rows_dyn) */
#define DKSS_ROWS_CLUSTER 3     /* row phase as one thread-block-cluster kernel (k_rows) */
#define DKSS_PASS_AUTO 0
#define DKSS_PASS_CTA 1         /* column pass: one CTA per column tile */
#define DKSS_PASS_WARP 2        /* column pass: warp per column */
#define DKSS_PASS_SPLIT 3       /* column DFT kernel + elementwise twiddle kernel */
#define DKSS_TWIDDLE_AUTO 0     /* tensor cores where the plan allows (m in {16, 32}, L = 4, Proth p) */
#define DKSS_TWIDDLE_CUDA 1     /* twiddle ring products on the CUDA cores (IMAD.WIDE carry chains) */
#define DKSS_TWIDDLE_TENSOR 2   /* twiddle ring products on the tensor cores (tcgen05 kind::i8) */
typedef struct {
  int32_t row_phase; /* DKSS_ROWS_*; ignored by plans that are not two-level */
  int32_t pass_kind; /* DKSS_PASS_* */
  int32_t twiddle;   /* DKSS_TWIDDLE_*: the engine of the table-twiddle ring products */
} dkss_plan_opts;

/* plan lifetime -------------------------------------------------------------------- */
int dkss_plan_create(const dkss_plan_desc* desc, int device, dkss_plan** out);
int dkss_plan_create_ex(const dkss_plan_desc* desc, const dkss_plan_opts* opts, int device, dkss_plan** out);
void dkss_plan_destroy(dkss_plan* plan);
int dkss_plan_get_info(const dkss_plan* plan, dkss_plan_info* out);
const char* dkss_last_error(void);
int dkss_version(void);
/* kernels this process has launched through the library so far (a CUDA-graph replay counts
 * each of its kernel nodes); instrumentation for benchmarks (bench.py "gpu_launches") */
int64_t dkss_kernel_launches(void);
/* device bytes one multiply of host operands holds for a plan of this shape (twiddle tables,
 * the two polynomials, operand staging, operands, product, decode scratch): the memory figure
 * dmul records in the caller's ScratchArena (cf. bigmul/dkss.py:538-539).  Needs no GPU; -1 for a
 * bad shape. */
int64_t dkss_footprint_bytes(int64_t N, int32_t M, int32_t m, int32_t L);

/* Page-locked host buffers from a library pool (recycled by size).  A product buffer `c` from
 * here receives the products of dkss_mul_digits / dkss_mul_batch_digits straight from the device
 * (no staging copy); dkss_host_free returns it to the pool. */
int dkss_host_alloc(size_t bytes, void** out);
void dkss_host_free(void* p);

/* dmul (bigmul/dkss.py:520-548) for operands below 2^N: c = a * b.
 * Host buffers; na, nb <= operand_limbs; nc limbs are written (zero padded); the call
 * fails with DKSS_ERANGE if the product does not fit nc limbs. */
int dkss_mul(dkss_plan* plan, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint32_t* c, size_t nc);

/* dmul with operands given as little-endian radix-2^digit_bits digit strings, one digit
 * per uint32 (8 <= digit_bits <= 32) -- e.g. the 30-bit digits of a CPython int, so the
 * host does no radix conversion (the device repacks them to 32-bit limbs).  The product
 * is written as nc 32-bit limbs, as dkss_mul. */
int dkss_mul_digits(dkss_plan* plan, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int digit_bits,
                    uint32_t* c, size_t nc);
/* OR into digit_bits when every digit is known to be < 2^digit_bits (e.g. a CPython int's
 * digits): the library then skips its scan of the digit strings */
#define DKSS_DIGITS_TRUSTED 0x100
/* batched form: pair i is a[i] (na[i] digits) x b[i] (nb[i] digits); c is batch x nc limbs */
int dkss_mul_batch_digits(dkss_plan* plan, int batch, const uint32_t* const* a, const size_t* na,
                          const uint32_t* const* b, const size_t* nb, int digit_bits, uint32_t* c, size_t nc);

/* batched independent products sharing one plan (config 3): a, b are batch x n_limbs,
 * c is batch x nc.  Host buffers. */
int dkss_mul_batch(dkss_plan* plan, int batch, const uint32_t* a, const uint32_t* b, size_t n_limbs, uint32_t* c,
                   size_t nc);

/* device-resident variant: a_dev, b_dev, c_dev are device pointers with the same shapes,
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Stream-ordered; replays a
 * cached CUDA graph per (pointers, batch, sizes).  b_dev == NULL squares a (one forward
 * transform instead of two). */
int dkss_mul_device(dkss_plan* plan, int batch, const uint32_t* a_dev, const uint32_t* b_dev, size_t n_limbs,
                    uint32_t* c_dev, size_t nc, void* stream);

/* per-launch profile of one device multiply (same launches as dkss_mul_device, not graphed):
 * a CUDA event is recorded on `stream` after every kernel; for launch i, kinds[i] is a
 * DKSS_K_* id, ms[i] its event-to-event duration, work[i] the algorithmic 32x32->64 limb
 * products it performs (ring products x m^2 L^2) -- for DKSS_K_TWIDDLE_TC the
 * int8 operations of its byte GEMM on the live rows (rows x 16m x 16m x 2) -- and bytes[i] the
 * stage-boundary HBM bytes of the §8(d) model.  c_dev receives the product (product_limbs). */
#define DKSS_K_ENCODE 0
#define DKSS_K_FWD_PASS 1
#define DKSS_K_BOTTOM 2
#define DKSS_K_INV_PASS 3
#define DKSS_K_DECODE1 4
#define DKSS_K_DECODE2 5
#define DKSS_K_ROWS 7 /* row phase in one cluster kernel (levels >= 1, pointwise, inverse levels >= 1) */
#define DKSS_K_TRANSPOSE 6
#define DKSS_K_TWIDDLE_TC 8 /* one level's table-twiddle ring products on the tensor cores */
int dkss_profile_device(dkss_plan* plan, int batch, const uint32_t* a_dev, const uint32_t* b_dev, size_t n_limbs,
                        uint32_t* c_dev, void* stream, int max_launches, int32_t* kinds, float* ms, int64_t* work,
                        int64_t* bytes, int* n_launches);

/* four-step split of ONE multiply over `world` GPUs (the reference's radix
 * split of dkss_fft, bigmul/dkss.py:465-495).  E = 2m, mu0 = 2M/E; an element is m*L limbs.
 * Rank r owns the global columns [r*C, (r+1)*C), C = mu0/world, of the first transform level,
 * stored [E][C] per polynomial; after the exchange rank h owns the rows [h*R, (h+1)*R),
 * R = E/world, stored [R][mu0] per polynomial.  world: power of 2, <= E, dividing mu0.
 * All buffers are device pointers; every call is stream-ordered; the exchange itself (an
 * all-to-all of world blocks of block_words/world limbs per polynomial) is the caller's, e.g.
 * NCCL through torch.distributed (paper_1503_04955_b200/fourstep.py). */
typedef struct {
  int64_t cols;        /* C, first-level columns per rank */
  int64_t rows;        /* R, rows per rank after the exchange */
  int64_t elem_words;  /* m*L */
  int64_t block_words; /* one polynomial's share per rank: poly_words / world */
  int64_t decode_seg;  /* distributed decode (u = 32): limbs per run segment; a rank writes
                          (2m + 1) segments of 64-bit window sums; 0 when u != 32 */
} dkss_fs_layout;
int dkss_fs_layout_get(const dkss_plan* plan, int world, dkss_fs_layout* out);
/* encode (bigmul/dkss.py:381-398) fused with the first forward level (column DFTs + twiddles,
 * bigmul/dkss.py:471-492) of a and b over this rank's columns: x = [2][E][C] elements */
int dkss_fs_columns_fwd(dkss_plan* plan, int rank, int world, const uint32_t* a_dev, const uint32_t* b_dev,
                        size_t n_limbs, uint32_t* x_dev, void* stream);
/* rows phase: deeper forward levels of a and b (bigmul/dkss.py:493-495), pointwise r_mul
 * (bigmul/dkss.py:544-545), deeper inverse levels of the product: z = [2][R][mu0] elements
 * (a rows then b rows); the product rows are left in z[0] */
int dkss_fs_rows(dkss_plan* plan, int world, uint32_t* z_dev, void* stream);
/* last inverse level (columns) of the product with the 1/2M scaling (bigmul/dkss.py:507):
 * x = [E][C] elements of this rank's columns */
int dkss_fs_columns_inv(dkss_plan* plan, int rank, int world, uint32_t* x_dev, void* stream);
/* distributed decode (u = 32): after dkss_fs_columns_inv, every rank turns its columns into
 * the per-limb window sums of its logical runs, s_out = uint64[2m + 1][decode_seg]
 * (bigmul/dkss.py:498-513 restricted to the rank's coefficients); rank 0 gathers the world's
 * segments, parts = uint64[world][2m + 1][decode_seg], adds the overlapping runs and
 * resolves the carries into nc >= product_limbs limbs */
int dkss_fs_decode_partial(dkss_plan* plan, int rank, int world, const uint32_t* x_dev, uint64_t* s_out_dev,
                           void* stream);
int dkss_fs_decode_finish(dkss_plan* plan, int world, const uint64_t* parts_dev, uint32_t* out_dev, size_t nc,
                          void* stream);
/* the same two phases with the exchange fused into their stores: instead
 * of this rank's x (resp. its product rows in z) each output element is written straight into
 * the buffer of the rank that owns it next -- z_peers[h] = rank h's z = [2][R][mu0] rows,
 * x_peers[r] = rank r's x = [E][C] columns of the product -- through device-visible peer base
 * pointers (a device array of `world` uint64 addresses: CUDA IPC mappings of the other GPUs'
 * buffers over NVLink, or plain pointers for ranks emulated on one GPU).  No all-to-all and no
 * re-layout; the caller orders the phases across ranks (a stream-ordered barrier such as a
 * one-element NCCL all-reduce).  The rows phase needs >= 2 transform levels.  x_dev of the
 * first call is this rank's [2][E][C] scratch: elements whose table twiddles the tensor cores
 * apply pass through it (the tensor-core kernel stores them to their owners). */
int dkss_fs_columns_fwd_peer(dkss_plan* plan, int rank, int world, const uint32_t* a_dev, const uint32_t* b_dev,
                             size_t n_limbs, uint32_t* x_dev, const uint64_t* z_peers_dev, void* stream);
int dkss_fs_rows_peer(dkss_plan* plan, int rank, int world, uint32_t* z_dev, const uint64_t* x_peers_dev,
                      void* stream);
/* device buffers shareable with the other ranks' processes (cudaMalloc + CUDA IPC): handle is a
 * 64-byte cudaIpcMemHandle_t; dkss_ipc_open maps another process's buffer on `device` */
int dkss_ipc_alloc(int device, size_t bytes, void** dptr, void* handle);
int dkss_ipc_open(int device, const void* handle, void** dptr);
int dkss_ipc_close(void* dptr);
int dkss_ipc_free(void* dptr);
/* exchange re-layout: src [n][A][B][run_words] -> dst [n][B][A][run_words] (16-byte aligned,
 * run_words a multiple of 4, n*A*B <= 65535) */
int dkss_block_transpose(dkss_plan* plan, const uint32_t* src_dev, uint32_t* dst_dev, int n, int A, int B,
                         int64_t run_words, void* stream);
/* dkss_decode (bigmul/dkss.py:498-513) on the device: v = the scaled inverse transform as
 * left by the device pipeline (full [E][mu0] layout); nc >= product_limbs limbs written */
int dkss_decode_device(dkss_plan* plan, const uint32_t* v_dev, uint32_t* out_dev, size_t nc, void* stream);

/* Lucas-Lehmer iterations (bigmul/bench.py:197-217) on the device: `iters` times
 * s <- (s^2 - 2) mod (2^p - 1), canonical in [0, 2^p - 1) (mersenne_reduce, :187-194),
 * each square through the DKSS pipeline in squaring mode.  s: host, ns >= ceil(p/32) limbs,
 * in and out; requires 2 <= p <= N of the plan. */
int dkss_lucas_lehmer(dkss_plan* plan, int64_t p, int64_t iters, uint32_t* s, size_t ns);

/* stage entry points for parity checks (host buffers) ------------------------------ */
/* dkss_encode, bigmul/dkss.py:381-398: poly = uint32[2M][m][L] */
int dkss_encode_host(dkss_plan* plan, const uint32_t* a, size_t na, uint32_t* poly);
/* dkss_fft, bigmul/dkss.py:443-495: count polynomials transformed in place (natural order) */
int dkss_fft_host(dkss_plan* plan, uint32_t* polys, int count);
/* r_mul, bigmul/dkss.py:401-420: count ring products out[i] = x[i]*y[i] (count x m x L) */
int dkss_rmul_host(dkss_plan* plan, const uint32_t* x, const uint32_t* y, uint32_t* out, size_t count);
/* dkss_decode, bigmul/dkss.py:498-513: v = forward transform of the product polynomial
 * (natural order, still scaled by 2M); out gets nout limbs of the integer */
int dkss_decode_host(dkss_plan* plan, const uint32_t* v, uint32_t* out, size_t nout);

#ifdef __cplusplus
}
#endif
#endif /* DKSS_H */
