// dkss_capi.cu -- libdkss: plan upload, device workspace, launch sequence, C ABI.
// See include/dkss.h for the contract and DESIGN.md for the kernel/roofline story.
#include <cuda.h>  // CUtensorMap types only: the encoder is fetched through cudaGetDriverEntryPoint
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <chrono>
#include <tuple>
#include <vector>

#include "../../include/dkss.h"
#define DKSS_COMMON_KERNELS
#include "dkss_table.cuh"

using namespace dkss;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUCHK(expr)                                                                              \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess) return fail(DKSS_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// Experiment switches (timing studies, kernel A/B runs) exist only in DKSS_VARIANT builds
// (paper_1503_04955_b200/build.py defines DKSS_EXPERIMENTS there); the product library reads
// no environment variables.
#ifdef DKSS_EXPERIMENTS
#define DKSS_KNOB(name) getenv(name)
#else
#define DKSS_KNOB(name) ((const char*)nullptr)
#endif

bool knob_on(const char* v) { return v && *v && *v != '0'; }

// Every stream of this library is non-blocking, so nothing orders it after work on the legacy
// default stream -- and a synchronous cudaMemcpy from pageable host memory may return once the
// source is staged, before the DMA has landed (CUDA "API synchronization behavior"), as may a
// cudaMemset.  Plan tables, schedules and counters are therefore uploaded on a private stream that
// is synchronized before returning (legal while another stream of the thread is being captured,
// unlike a device-wide synchronize).  Without it a plan's twiddle table was occasionally read
// half-uploaded: about one fresh large plan in a few hundred gave products that were wrong in
// every bit until the plan was rebuilt -- found by tools/soak.py.  src == nullptr: zero fill.
cudaError_t upload_sync(void* dst, const void* src, size_t bytes) {
  constexpr int kMaxDev = 64;
  static thread_local cudaStream_t up[kMaxDev] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!up[dev] && (e = cudaStreamCreateWithFlags(&up[dev], cudaStreamNonBlocking)) != cudaSuccess) return e;
  e = src ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, up[dev]) : cudaMemsetAsync(dst, 0, bytes, up[dev]);
  if (e == cudaSuccess) e = cudaStreamSynchronize(up[dev]);
  return e;
}

// kernels this library launched (graph replays add their kernel nodes), for dkss_kernel_launches()
std::atomic<long long> g_launches{0};
// set while a stream of this thread is being captured into a graph: launches then become graph
// nodes and are counted when the graph is replayed
thread_local bool tl_capturing = false;
inline void count_launch() {
  if (!tl_capturing) g_launches.fetch_add(1, std::memory_order_relaxed);
}

struct CaptureScope {
  CaptureScope() { tl_capturing = true; }
  ~CaptureScope() { tl_capturing = false; }
};

int graph_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (n && cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// Executable graphs keyed by K, least recently used evicted beyond `cap`.  Each entry keeps an
// event recorded after its last replay, so an evicted graph is destroyed only once its last
// replay has finished.
template <class K>
struct GraphLru {
  struct Ent {
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;
    int kernels = 0;
    unsigned long long stamp = 0;
  };
  explicit GraphLru(size_t cap_) : cap(cap_) {}
  std::map<K, Ent> m;
  unsigned long long clock = 0;
  size_t cap;
  Ent* find(const K& k) {
    auto it = m.find(k);
    if (it == m.end()) return nullptr;
    it->second.stamp = ++clock;
    return &it->second;
  }
  static void destroy(Ent& e) {
    if (e.done) {
      cudaEventSynchronize(e.done);
      cudaEventDestroy(e.done);
    }
    if (e.exec) cudaGraphExecDestroy(e.exec);
  }
  // instantiate g (consumed) under key k; returns nullptr and sets *err on failure
  Ent* put(const K& k, cudaGraph_t g, cudaError_t* err) {
    while (m.size() >= cap) {
      auto old = m.begin();
      for (auto it = m.begin(); it != m.end(); ++it)
        if (it->second.stamp < old->second.stamp) old = it;
      destroy(old->second);
      m.erase(old);
    }
    Ent e;
    e.kernels = graph_kernel_nodes(g);
    cudaError_t r = cudaGraphInstantiate(&e.exec, g, 0);
    cudaGraphDestroy(g);
    if (r == cudaSuccess) r = cudaEventCreateWithFlags(&e.done, cudaEventDisableTiming);
    if (r != cudaSuccess) {
      if (e.exec) cudaGraphExecDestroy(e.exec);
      *err = r;
      return nullptr;
    }
    e.stamp = ++clock;
    return &(m[k] = e);
  }
  cudaError_t launch(Ent* e, cudaStream_t s) {
    cudaError_t r = cudaGraphLaunch(e->exec, s);
    if (r == cudaSuccess) r = cudaEventRecord(e->done, s);
    if (r == cudaSuccess) g_launches.fetch_add(e->kernels, std::memory_order_relaxed);
    return r;
  }
  void clear() {
    for (auto& kv : m) destroy(kv.second);
    m.clear();
  }
  size_t size() const { return m.size(); }
};

int ilog2i(long long v) {
  int k = 0;
  while ((1LL << k) < v) ++k;
  return k;
}

// ---- host multiprecision for the plan constants ----------------------------------
using Limbs = std::vector<uint32_t>;

int cmp(const Limbs& a, const Limbs& b) {
  for (int i = (int)a.size() - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
  return 0;
}
void sub_inplace(Limbs& a, const Limbs& b) {
  int64_t br = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    int64_t x = (int64_t)a[i] - b[i] + br;
    a[i] = (uint32_t)x;
    br = x >> 32;
  }
}
// a = 2a mod p  (a < p)
void dbl_mod(Limbs& a, const Limbs& p) {
  uint32_t carry = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    uint32_t nc = a[i] >> 31;
    a[i] = (a[i] << 1) | carry;
    carry = nc;
  }
  if (carry || cmp(a, p) >= 0) sub_inplace(a, p);
}
// a = a/2 mod p  (p odd)
void half_mod(Limbs& a, const Limbs& p) {
  uint32_t top = 0;
  if (a[0] & 1) {
    uint64_t c = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      c += (uint64_t)a[i] + p[i];
      a[i] = (uint32_t)c;
      c >>= 32;
    }
    top = (uint32_t)c;
  }
  for (size_t i = 0; i < a.size(); ++i) {
    uint32_t hi = i + 1 < a.size() ? a[i + 1] : top;
    a[i] = (a[i] >> 1) | (hi << 31);
  }
}

// ---- kernel table per (m, L): instantiated in dkss_inst_m{8,16,32}.cu ----------------
bool lookup(int m, int L, KTable* out) {
  KTable t{};
#define DKSS_CASE(MM, L_) \
  if (m == MM && L == L_) t = dkss_table_m##MM##_L##L_();
  DKSS_FOR_EACH_INST(DKSS_CASE)
#undef DKSS_CASE
  *out = t;
  return t.fwd != nullptr;
}

}  // namespace

struct GraphKey {
  int batch;
  const void* a;
  const void* b;
  void* c;
  size_t nl, nc;
  bool operator<(const GraphKey& o) const {
    return std::tie(batch, a, b, c, nl, nc) < std::tie(o.batch, o.a, o.b, o.c, o.nl, o.nc);
  }
};

// device-pointer graphs kept per plan: a caller cycling through more buffer triples than this
// re-captures (about 20 us for a two-level plan) instead of growing the cache without bound
constexpr size_t kGraphCacheCap = 16;

// tensor-core twiddle schedule of one (level, polynomials per launch): tiles of <= 128
// twiddled elements sharing a table row s, each tile's entries in a 128-slot block
struct TcSched {
  uint32_t* d_tiles = nullptr;    // [ntiles][3] s, first entry, count
  uint32_t* d_entries = nullptr;  // [ntiles][128] (element << 6) | alpha shift
  int ntiles = 0;
  long long twiddled = 0;         // elements with s != 0
};

struct dkss_plan {
  int device = 0;
  long long N = 0;
  int M = 0, m = 0, u = 0, L = 0;
  int levels = 0, base_len = 0, logE = 0, logb = 0, log_top_mu = 0;
  long long poly_words = 0, op_limbs = 0, prod_limbs = 0;
  long long twiddles = 0;
  ModCtx mc{};
  KTable kt{};
  uint32_t* d_tw = nullptr;   // Montgomery-form rho table [M/m][m][L]
  uint32_t* d_twr = nullptr;  // twiddle rows [M/m][2m][L]: Montgomery-form rho^s, then W_s
  uint32_t* d_twr_s = nullptr;  // the same rows times (2M)^-1 R: the last inverse level scales for free
  int grid_pass = 0, grid_bot = 0;  // persistent grid sizes (SMs x resident CTAs)
  int grid_pass_do = 0;             // DFT-only passes (kt.fwd_do / inv_do), 0 = not used
  int grid_fw = 0, grid_iw = 0;     // warp-per-column kernels (0 = not used)
  int grid_dft = 0, grid_tw = 0;    // split passes (column DFT kernel + elementwise twiddles)
  int pass_mode = 0;                // 0 auto, 1 CTA-fused, 2 warp-fused, 3 split
  int rows_cs = 0;                  // >0: row phase in one cluster kernel (k_rows, cluster size)
  int dyn_grid = 0;                 // >0: row phase as one persistent dependency-driven kernel
  unsigned* d_dyn = nullptr;        // its ticket + per-row counters (cap_batch rows)
  unsigned long long* d_sglob = nullptr;  // per-limb window sums of a distributed decode
  unsigned* d_tick = nullptr;       // per-launch tile tickets of the CTA kernels, kTickSlots x 2
  bool tc = false;                  // table twiddles on the tensor cores (dkss_tc.cuh) available
  bool tc_forced = false;           // DKSS_TWIDDLE_TENSOR: every full-layout launch uses them
  int tc_grid = 0;                  // SMs (one tensor-core CTA per SM)
  uint32_t tc_p3 = 0;               // p = 1 + tc_p3 * 2^96
  std::map<const void*, TcTensorMap> tc_tmaps;  // TMA descriptors of the element buffers seen (tc_tensor_map)
  uint8_t* d_vtab = nullptr;        // V tables of d_twr rows, [M/m][2m-1][16][16]
  uint8_t* d_vtab_s = nullptr;      // of the pre-scaled rows d_twr_s (last inverse level)
  std::map<std::tuple<int, long long, bool, int, int>, TcSched> tc_sched;  // by TcLayout
  int tick_next = 0;
  bool dyn_tiles = true;            // DKSS_NO_DYNTILES=1: static round-robin tiles
  void (*rows_fn)(RowsArgs, ModCtx) = nullptr;
  // workspace
  int cap_batch = 0;
  uint32_t* d_poly = nullptr;  // 2 * cap_batch polynomials
  uint32_t* d_ops = nullptr;   // 2 * cap_batch operands (host API staging)
  uint32_t* d_prod = nullptr;  // cap_batch products
  uint32_t* d_gmask = nullptr;
  uint32_t* d_pmask = nullptr;
  uint32_t* d_bstat = nullptr;
  uint32_t* h_pin = nullptr;   // pinned staging
  uint32_t* d_stage = nullptr; // device copy of radix-2^k operand digits (dkss_mul_digits)
  size_t stage_words = 0;
  size_t h_pin_words = 0;
  size_t ws_bytes = 0;
  cudaStream_t stream = nullptr;
  // host digits path, one product: operand transfers on their own stream so b's staging and H2D
  // overlap a's first transform level (run_digits_split)
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_ops[2] = {nullptr, nullptr};
  // replayed multiplies: device-pointer entry (keyed by the caller's buffers), Lucas-Lehmer
  // steps (p, iterations per graph), host digits path (batch, square, digit bits)
  GraphLru<GraphKey> graphs{kGraphCacheCap};
  GraphLru<std::pair<long long, int>> ll_graphs{8};
  GraphLru<std::tuple<int, bool, int>> dgraphs{8};
  std::mutex mu;
  struct Prof {
    static constexpr int kMax = 64;
    cudaEvent_t ev[kMax + 1];
    int kind[kMax];
    long long work[kMax], bytes[kMax];
    int n = 0;
  }* prof = nullptr;  // non-null only inside dkss_profile_device
};

namespace {

int dec_blocks(const dkss_plan* P) { return (int)((P->prod_limbs + kDecThreads - 1) / kDecThreads); }

void free_ws(dkss_plan* P) {
  cudaFree(P->d_poly);
  cudaFree(P->d_ops);
  cudaFree(P->d_prod);
  cudaFree(P->d_gmask);
  cudaFree(P->d_pmask);
  cudaFree(P->d_bstat);
  cudaFree(P->d_dyn);
  P->d_dyn = nullptr;
  P->d_poly = P->d_ops = P->d_prod = P->d_gmask = P->d_pmask = P->d_bstat = nullptr;
  P->graphs.clear();
  P->ll_graphs.clear();
  P->dgraphs.clear();
  P->cap_batch = 0;
  P->ws_bytes = 0;
}

int ensure_ws(dkss_plan* P, int batch) {
  if (batch <= P->cap_batch) return 0;
  free_ws(P);
  const size_t poly_b = (size_t)P->poly_words * 4;
  const size_t nwarps = (size_t)dec_blocks(P) * kDecWarps;
  CUCHK(cudaMalloc(&P->d_poly, 2 * (size_t)batch * poly_b));
  CUCHK(cudaMalloc(&P->d_ops, 2 * (size_t)batch * P->op_limbs * 4));
  CUCHK(cudaMalloc(&P->d_prod, (size_t)batch * P->prod_limbs * 4));
  CUCHK(cudaMalloc(&P->d_gmask, (size_t)batch * nwarps * 4));
  CUCHK(cudaMalloc(&P->d_pmask, (size_t)batch * nwarps * 4));
  CUCHK(cudaMalloc(&P->d_bstat, (size_t)batch * dec_blocks(P) * 4));
  CUCHK(cudaMalloc(&P->d_dyn, (4 + 2 * (size_t)batch * 2 * P->m) * 4));
  CUCHK(upload_sync(P->d_dyn, nullptr, (4 + 2 * (size_t)batch * 2 * P->m) * 4));
  P->cap_batch = batch;
  P->ws_bytes = 2 * (size_t)batch * poly_b + 2 * (size_t)batch * P->op_limbs * 4 + (size_t)batch * P->prod_limbs * 4 +
                (size_t)batch * nwarps * 8 + (size_t)batch * dec_blocks(P) * 4;
  return 0;
}

int ensure_pin(dkss_plan* P, size_t words) {
  if (words <= P->h_pin_words) return 0;
  P->dgraphs.clear();  // they copy to/from h_pin
  if (P->h_pin) cudaFreeHost(P->h_pin);
  P->h_pin = nullptr;
  CUCHK(cudaMallocHost(&P->h_pin, words * 4));
  P->h_pin_words = words;
  return 0;
}

// per-launch accounting hook (kinds: see dkss.h DKSS_K_*)
void mark(dkss_plan* P, cudaStream_t s, int kind, long long work, long long bytes) {
  auto* pr = P->prof;
  if (!pr || pr->n >= dkss_plan::Prof::kMax) return;
  pr->kind[pr->n] = kind;
  pr->work[pr->n] = work;
  pr->bytes[pr->n] = bytes;
  cudaEventRecord(pr->ev[++pr->n], s);
}

long long rp_work(const dkss_plan* P, long long ring_products) { return ring_products * P->m * P->m * P->L * P->L; }

long long level_twiddles(const dkss_plan* P, int lv) {
  const long long E = 2LL * P->m;
  const long long mu = (2LL * P->M) >> (P->logE * (lv + 1));
  return (1LL << (P->logE * lv)) * (E - 1) * (mu - 1);
}

size_t smem_pass(const dkss_plan* P) { return P->kt.smem_pass; }
size_t smem_two(const dkss_plan* P) { return P->kt.smem_bot; }

// kernel launch with programmatic dependent launch allowed (the kernels call griddep_wait()
// before touching their predecessor's output); DKSS_NO_PDL=1 turns it off
bool pdl_enabled() {
  static const bool on = [] {
    return !knob_on(DKSS_KNOB("DKSS_NO_PDL"));
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
  count_launch();
}

// --- launch helpers (all stream-ordered) ---------------------------------------------
// ticket counter pair for the next CTA-kernel launch (consecutive launches get different
// slots, so a PDL-overlapped successor never shares one; each launch re-zeroes its own)
constexpr int kTickSlots = 64;
// Only worth it with several tiles per resident CTA: below that the ticket round trip before
// each prefetch costs more than the balance gains (2^20, 1.7 tiles per CTA: +4%; batch
// 1024 x 2^18: -9%; the 2^24 inverse, 3.5 tiles per CTA: -1.5%)
unsigned* next_tick(dkss_plan* P, long long tiles = 1LL << 62, int grid = 1) {
  if (!P->dyn_tiles || !P->d_tick || tiles < 3LL * grid) return nullptr;
  unsigned* c = P->d_tick + 2 * (P->tick_next % kTickSlots);
  ++P->tick_next;
  return c;
}

int launch_encode(dkss_plan* P, const uint32_t* ops, long long na, uint32_t* poly, int npoly, cudaStream_t s) {
  EncodeArgs A{ops, na, poly, P->poly_words, npoly, P->M, P->m, P->L, P->u};
  const long long total = 2LL * P->M * P->m * npoly;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  launch_k(k_encode, dim3(blocks), dim3(256), 0, s, A);
  CUCHK(cudaGetLastError());
  mark(P, s, DKSS_K_ENCODE, 0, npoly * (P->op_limbs * 4 + P->poly_words * 4));
  return 0;
}

// pass implementation for a launch over `cols` columns: 1 CTA-fused, 2 warp-fused, 3 split
int pass_kind(const dkss_plan* P, long long cols) {
  if (P->pass_mode) return (P->pass_mode == 3 && !P->grid_dft) ? 1 : (P->pass_mode == 2 && !P->grid_fw) ? 1 : P->pass_mode;
  // with ticketed tiles the CTA-wide kernel is at least as fast as warp-per-column everywhere
  // (batch 1024 x 2^18 forward: 5.76 vs 5.81 ms); without them large launches prefer warps
  if (!P->dyn_tiles && P->grid_fw && cols >= 4LL * P->grid_fw * kWarpsPerCta) return 2;
  return 1;
}

void launch_dft(dkss_plan* P, const PassArgs& A, long long cols, cudaStream_t s) {
  const int g = (int)std::min<long long>(P->grid_dft, (cols + kWarpsPerCta - 1) / kWarpsPerCta);
  launch_k(P->kt.dft, dim3(g), dim3(kWarpsPerCta * 32), P->kt.smem_dft, s, A, P->mc);
}

void launch_tw(dkss_plan* P, const PassArgs& A, long long cols, cudaStream_t s) {
  const long long items = cols * 2 * P->m * (P->m / 2);  // T = 2 outputs per item
  const int g = (int)std::min<long long>(P->grid_tw, (items + 255) / 256);
  launch_k(P->kt.tw, dim3(g), dim3(256), 0, s, A, P->mc);
}

// layout of the polynomials a pass launch walks (see PassArgs): the whole transform
// (full_geom), the local column block of a sharded first level, or the rows of a
// sharded second phase (four-step split, dkss_fs_*)
struct Geom {
  long long poly_words;  // words per polynomial in this layout
  int log_cpp;           // log2 columns per polynomial
  long long l_off;       // global column offset (first level of a column shard)
  int log_mu0;           // column stride at level 0 in this layout (-1: 2M/2m)
  // fused four-step exchange (PassArgs::peer_mode): applied to the last level the call runs
  const unsigned long long* peer = nullptr;
  int peer_mode = 0, peer_log_r = 0, peer_log_c = 0, peer_log_mu0 = 0;
  long long peer_row0 = 0;
};

Geom full_geom(const dkss_plan* P) { return Geom{P->poly_words, P->log_top_mu, 0, -1}; }

void set_peer(PassArgs& A, const Geom& g) {
  A.peer = g.peer;
  A.peer_mode = g.peer_mode;
  A.peer_log_r = g.peer_log_r;
  A.peer_log_c = g.peer_log_c;
  A.peer_log_mu0 = g.peer_log_mu0;
  A.peer_row0 = g.peer_row0;
}

PassArgs pass_args(const dkss_plan* P, const Geom& g, uint32_t* poly, int npoly, int lv) {
  PassArgs A{};
  A.poly = poly;
  A.poly_words = g.poly_words;
  // column stride at level lv: mu_lv = 2M / (2m)^(lv+1)
  A.log_mu = (lv == 0 && g.log_mu0 >= 0) ? g.log_mu0 : ilog2i(2LL * P->M) - P->logE * (lv + 1);
  A.log_top_mu = P->log_top_mu;
  A.log_cpp = g.log_cpp;
  A.l_off = g.l_off;
  A.log_mu_enc = P->log_top_mu;
  A.base_pow = 1LL << (P->logE * lv);
  A.twr = P->d_twr;
  A.scale = 0;
  A.total_cols = (long long)npoly << g.log_cpp;
  A.wpc = 1;
  return A;
}

// Which elements one tensor-core launch covers (the layouts of the pass kernels):
//   full layout, level 0: `count` polynomials of 2M elements;
//   rows layout, level >= 1: `count` rows of mu0 = M/m elements (a full-layout launch over n
//     polynomials at level >= 1 is the rows layout over n E rows: levels >= 1 act inside a row);
//   columns layout, level 0 (four-step split): `count` polynomials of E x C
//     elements, this rank's columns [col_rank C, (col_rank + 1) C), C = mu0 / col_world.
struct TcLayout {
  int lv = 0;
  long long count = 0;
  bool rows = false;
  int col_rank = 0, col_world = 0;
};

TcLayout tc_full(const dkss_plan* P, int lv, int npoly) {
  TcLayout t;
  t.lv = lv;
  t.count = npoly;
  if (lv >= 1) {
    t.rows = true;
    t.count = (long long)npoly * 2 * P->m;
  }
  return t;
}

// tensor-core twiddle schedule of one launch (built on the host once per layout): every element
// with a table twiddle, e = j l (2m)^lv, s = e mod (M/m) != 0, grouped by s into tiles of <= 128
int tc_sched(dkss_plan* P, const TcLayout& lay, const TcSched** out) {
  const auto key = std::make_tuple(lay.lv, lay.count, lay.rows, lay.col_rank, lay.col_world);
  auto it = P->tc_sched.find(key);
  if (it != P->tc_sched.end()) {
    *out = &it->second;
    return 0;
  }
  const long long E = 2LL * P->m, twoM = 2LL * P->M, mu_top = 1LL << P->log_top_mu, mu0 = mu_top;
  const int lv = lay.lv;
  const int log_mu = ilog2i(twoM) - P->logE * (lv + 1);
  const long long mu = 1LL << log_mu, base_pow = 1LL << (P->logE * lv);
  std::vector<std::vector<uint32_t>> groups((size_t)mu_top);
  long long total = 0;
  auto add = [&](long long el, long long j, long long l) {
    const long long e = j * l * base_pow;
    const long long sr = e & (mu_top - 1);
    if (!sr) return;
    const long long r = (e >> P->log_top_mu) & (E - 1);
    groups[(size_t)sr].push_back((uint32_t)(el << 6 | r));
  };
  if (lay.rows) {
    total = lay.count * mu0;
    const long long inst = mu0 / (E * mu);
    if (total < (1LL << 26))
      for (long long u = 0; u < lay.count; ++u)
        for (long long in = 0; in < inst; ++in)
          for (long long j = 1; j < E; ++j)
            for (long long l = 1; l < mu; ++l) add(u * mu0 + (in << (log_mu + P->logE)) + (j << log_mu) + l, j, l);
  } else if (lay.col_world) {
    const long long C = mu0 / lay.col_world;
    total = lay.count * E * C;
    if (total < (1LL << 26))
      for (long long q = 0; q < lay.count; ++q)
        for (long long j = 1; j < E; ++j)
          for (long long c = 0; c < C; ++c) add(q * E * C + j * C + c, j, (long long)lay.col_rank * C + c);
  } else {
    total = lay.count * twoM;
    if (total < (1LL << 26))
      for (long long q = 0; q < lay.count; ++q)
        for (long long j = 1; j < E; ++j)
          for (long long l = 1; l < mu0; ++l) add(q * twoM + (j << P->log_top_mu) + l, j, l);
  }
  if (total >= (1LL << 26)) return fail(DKSS_EINVAL, "tensor-core schedule: too many elements");
  std::vector<uint32_t> tiles, entries;
  long long tw = 0;
  for (long long sr = 1; sr < mu_top; ++sr) {
    const auto& g = groups[(size_t)sr];
    tw += (long long)g.size();
    for (size_t k = 0; k < g.size(); k += kTcRows) {
      const size_t n = std::min<size_t>(kTcRows, g.size() - k);
      tiles.push_back((uint32_t)sr);
      tiles.push_back((uint32_t)entries.size());
      tiles.push_back((uint32_t)n);
      entries.insert(entries.end(), g.begin() + (long)k, g.begin() + (long)(k + n));
      entries.resize(entries.size() + (kTcRows - n), 0u);
    }
  }
  TcSched sc;
  sc.ntiles = (int)(tiles.size() / 3);
  sc.twiddled = tw;
  if (sc.ntiles) {
    CUCHK(cudaMalloc(&sc.d_tiles, tiles.size() * 4));
    CUCHK(cudaMalloc(&sc.d_entries, entries.size() * 4));
    CUCHK(upload_sync(sc.d_tiles, tiles.data(), tiles.size() * 4));
    CUCHK(upload_sync(sc.d_entries, entries.data(), entries.size() * 4));
  }
  *out = &(P->tc_sched[key] = sc);
  return 0;
}

// whether a launch over `elems` elements takes the tensor-core twiddles: always for m = 32; for
// m = 16 only from 2^17 elements per launch (2^20 x 2^20, 16384 elements: 96 vs 82 us -- two
// extra launches per level cost more than the faster products; the 1024 x 2^18 batch: 8.37 vs
// 11.36 ms)
constexpr long long kTcMinElems16 = 1LL << 17;
bool use_tc_elems(const dkss_plan* P, long long elems) {
  if (!P->tc) return false;
  return P->tc_forced || P->m >= 32 || elems >= kTcMinElems16;
}
bool use_tc(const dkss_plan* P, int npoly) { return use_tc_elems(P, (long long)npoly * 2 * P->M); }

// schedules a multiply of `batch` products will use, built before a stream capture starts
// (their device buffers cannot be allocated inside one)
int tc_prepare(dkss_plan* P, int batch, bool sq) {
  const TcSched* sc;
  int rc;
  for (int lv = 0; lv < P->levels; ++lv) {
    if (use_tc(P, (sq ? 1 : 2) * batch) && (rc = tc_sched(P, tc_full(P, lv, (sq ? 1 : 2) * batch), &sc))) return rc;
    if (use_tc(P, batch) && (rc = tc_sched(P, tc_full(P, lv, batch), &sc))) return rc;
  }
  return 0;
}

// the table twiddles of one launch on the tensor cores, in place (scaled: the last inverse
// level); with g->peer_mode == 1 (the fused four-step exchange of the first level) the products
// are stored into the row owners' buffers instead
// The tensor-core kernel gathers its element rows with TMA (cp.async.bulk.tensor ... tile::gather4):
// a 2-D byte tensor [rows][16 m] over the launch's elements, box 128 B x 1 row, 128-byte swizzle.
// The row bound is nominal (the schedule's entries index inside the caller's buffer).
int tc_tensor_map(dkss_plan* P, uint32_t* poly, TcTensorMap* out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (Encode)fn;
  }();
  if (!enc) return fail(DKSS_ECUDA, "cuTensorMapEncodeTiled is not available from this driver");
  static_assert(sizeof(TcTensorMap) == sizeof(CUtensorMap), "tensor map size");
  auto it = P->tc_tmaps.find(poly);
  if (it != P->tc_tmaps.end()) {
    *out = it->second;
    return 0;
  }
  const cuuint64_t row_bytes = (cuuint64_t)P->m * P->L * 4;
  const cuuint64_t gdim[2] = {row_bytes, (cuuint64_t)1 << 26};
  const cuuint64_t gstride[1] = {row_bytes};
  const cuuint32_t box[2] = {128, 1};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMap tm;
  const CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, poly, gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DKSS_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  memcpy(out, &tm, sizeof(tm));
  if (P->tc_tmaps.size() >= 64) P->tc_tmaps.clear();
  P->tc_tmaps[poly] = *out;
  return 0;
}

int launch_tc_layout(dkss_plan* P, uint32_t* poly, const TcLayout& lay, bool scaled, cudaStream_t s,
                     const Geom* peer = nullptr) {
  const TcSched* sc;
  int rc;
  if ((rc = tc_sched(P, lay, &sc))) return rc;
  if (!sc->ntiles) return 0;
  TcArgs A{};
  if ((rc = tc_tensor_map(P, poly, &A.tmap))) return rc;
  A.poly = poly;
  A.tiles = sc->d_tiles;
  A.entries = sc->d_entries;
  A.vtab = scaled ? P->d_vtab_s : P->d_vtab;
  A.ntiles = sc->ntiles;
  A.p3 = P->tc_p3;
  if (peer && peer->peer_mode == 1) {
    A.peer = peer->peer;
    A.peer_log_r = peer->peer_log_r;
    A.peer_log_c = peer->peer_log_c;
    A.peer_log_mu0 = peer->peer_log_mu0;
    A.peer_log_poly = P->logE + peer->peer_log_c;
    A.l_off = peer->l_off;
  }
  const int grid = std::min(sc->ntiles, P->tc_grid);
  launch_k(P->kt.tc, dim3(grid), dim3(kTcThreads), P->kt.smem_tc, s, A);
  CUCHK(cudaGetLastError());
  // work: the byte-GEMM's int8 operations on the live rows (rows x K x N x 2, K = 16m, N = 32m);
  // bytes: elements read and written once, one V table per tile
  mark(P, s, DKSS_K_TWIDDLE_TC, 2LL * sc->twiddled * (16LL * P->m) * (16LL * P->m),
       2LL * sc->twiddled * P->m * P->L * 4 + (long long)sc->ntiles * (long long)P->kt.tc_vbytes);
  return 0;
}

int launch_tc(dkss_plan* P, uint32_t* poly, int npoly, int lv, bool scaled, cudaStream_t s) {
  return launch_tc_layout(P, poly, tc_full(P, lv, npoly), scaled, s);
}

// the tensor-core layout of a pass launch over `npoly` polynomials of geometry g at level lv;
// false: CUDA-core twiddles (layout not covered, too few elements, or -- for the four-step
// layouts -- tiles too sparse: a rank holds 1/world of every twiddle group, and at an eighth of
// a tile per group the fixed cost per tile loses to the CUDA cores -- 2^26 on 8 ranks, first
// level, fill 0.125 / 0.062: 0.207 vs 0.194 ms forward, 0.228 vs 0.167 ms inverse -- while at a
// quarter it still wins: 2^24 on 2 ranks, inverse first level, fill 0.245: 0.118 vs 0.166 ms)
constexpr double kTcMinFill = 0.2;
bool tc_layout_of(dkss_plan* P, const Geom* g, int npoly, int lv, TcLayout* out) {
  if (!g) {
    *out = tc_full(P, lv, npoly);
    return use_tc(P, npoly);
  }
  bool ok = false;
  if (g->log_mu0 < 0 && lv >= 1) {  // rows layout: npoly rows of mu0 elements
    out->lv = lv;
    out->count = npoly;
    out->rows = true;
    ok = use_tc_elems(P, (long long)npoly << P->log_top_mu);
  } else if (g->log_mu0 >= 0 && lv == 0) {  // columns layout of a four-step rank
    out->lv = 0;
    out->count = npoly;
    out->col_world = 1 << (P->log_top_mu - g->log_cpp);
    out->col_rank = (int)(g->l_off >> g->log_cpp);
    ok = use_tc_elems(P, (long long)npoly * 2 * P->m << g->log_cpp);
  }
  if (!ok) return false;
  const TcSched* sc;
  if (tc_sched(P, *out, &sc)) {
    g_err.clear();
    return false;
  }
  return sc->ntiles == 0 || (double)sc->twiddled >= kTcMinFill * kTcRows * sc->ntiles;
}

// tc_npoly: polynomials the tensor-core decision is made for (default npoly); tc_launch = false
// leaves the table twiddles of these levels to the caller (one launch over more polynomials)
int launch_fwd_levels(dkss_plan* P, uint32_t* poly, int npoly, cudaStream_t s, const uint32_t* ops_a = nullptr,
                      const uint32_t* ops_b = nullptr, long long na = 0, int enc_split = 0, int lv_lo = 0,
                      int lv_hi = -1, const Geom* geom = nullptr, int tc_npoly = -1, bool tc_launch = true) {
  const Geom g = geom ? *geom : full_geom(P);
  if (lv_hi < 0) lv_hi = P->levels;
  const long long cols = (long long)npoly << g.log_cpp;
  const int grid = (int)std::min<long long>((cols + P->kt.cols - 1) / P->kt.cols, P->grid_pass);
  // ring products per level scale with the share of columns this launch covers
  const double share = (double)cols / ((double)npoly * (1LL << P->log_top_mu));
  for (int lv = lv_lo; lv < lv_hi; ++lv) {
    PassArgs A = pass_args(P, g, poly, npoly, lv);
    if (lv == 0 && ops_a) {
      A.ops_a = ops_a;
      A.ops_b = ops_b;
      A.na = na;
      A.enc_split = enc_split;
      A.u = P->u;
      A.M = P->M;
    }
    // auto mode: the first level (fused encode) runs the CTA-wide kernel, deeper levels may use
    // warp-per-column (batch 1024 x 2^18: forward 6.35 -> 5.95 ms)
    int kind = (lv == 0 && ops_a && !P->pass_mode) ? 1 : pass_kind(P, cols);
    if (g.peer_mode && lv == lv_hi - 1) {  // fused exchange: CTA kernel, stores to the owning ranks
      set_peer(A, g);
      kind = 1;
    }
    TcLayout tl;
    const bool tc = tc_layout_of(P, geom, tc_npoly > 0 ? tc_npoly : npoly, lv, &tl);
    if (tc) tc_layout_of(P, geom, npoly, lv, &tl);
    if (tc) {
      kind = 1;
      A.tw_skip = 1;
    }
    if (const char* fk = DKSS_KNOB("DKSS_FWD_KINDS")) {  // experiment: comma-separated kind per level
      int lvl = 0;
      for (const char* c = fk; *c; ++c) {
        if (*c == ',') ++lvl;
        else if (lvl == lv && *c >= '1' && *c <= '3') kind = *c - '0';
      }
      if ((kind == 2 && !P->grid_fw) || (kind == 3 && !P->grid_dft)) kind = 1;
    }
    if (kind == 3) {
      launch_dft(P, A, cols, s);
      CUCHK(cudaGetLastError());
      PassArgs B = A;
      B.ops_a = B.ops_b = nullptr;
      launch_tw(P, B, cols, s);
    } else if (kind == 2) {
      // warp-per-column only when every resident warp gets several columns (large batches);
      // small transforms keep the CTA-wide kernel, which spreads a column over 8 warps
      const long long wres = (long long)P->grid_fw * kWarpsPerCta;
      int wpc = 1;
      while (wpc < 8 && cols * wpc * 2 <= wres) wpc *= 2;
      A.wpc = wpc;
      const int gw = (int)std::min<long long>(P->grid_fw, (cols * wpc + kWarpsPerCta - 1) / kWarpsPerCta);
      launch_k(P->kt.fwd_w, dim3(gw), dim3(kWarpsPerCta * 32), P->kt.smem_fwd_w, s, A, P->mc);
    } else if (A.tw_skip && P->grid_pass_do) {  // DFT only: three CTAs per SM
      const long long tiles = (cols + P->kt.cols_do - 1) / P->kt.cols_do;
      const int gd = (int)std::min<long long>(tiles, P->grid_pass_do);
      A.ctr = next_tick(P, tiles, gd);
      launch_k(P->kt.fwd_do, dim3(gd), dim3(P->kt.nt), P->kt.smem_pass_do, s, A, P->mc);
    } else {
      A.ctr = next_tick(P, (cols + P->kt.cols - 1) / P->kt.cols, grid);
      launch_k(P->kt.fwd, dim3(grid), dim3(P->kt.nt), smem_pass(P), s, A, P->mc);
    }
    CUCHK(cudaGetLastError());
    mark(P, s, DKSS_K_FWD_PASS, tc ? 0 : (long long)(share * rp_work(P, npoly * level_twiddles(P, lv))),
         2LL * cols * 2 * P->m * P->m * P->L * 4);
    int rc;
    if (tc && tc_launch &&
        (rc = launch_tc_layout(P, poly, tl, false, s, (g.peer_mode && lv == lv_hi - 1) ? &g : nullptr)))
      return rc;
  }
  return 0;
}

int launch_inv_levels(dkss_plan* P, uint32_t* poly, int npoly, bool scale_last, cudaStream_t s, int lv_lo = 0,
                      int lv_hi = -1, const Geom* geom = nullptr) {
  const Geom g = geom ? *geom : full_geom(P);
  if (lv_hi < 0) lv_hi = P->levels;
  const long long cols = (long long)npoly << g.log_cpp;
  const int grid = (int)std::min<long long>((cols + P->kt.cols - 1) / P->kt.cols, P->grid_pass);
  const double share = (double)cols / ((double)npoly * (1LL << P->log_top_mu));
  for (int lv = lv_hi - 1; lv >= lv_lo; --lv) {
    PassArgs A = pass_args(P, g, poly, npoly, lv);
    A.scale = (lv == 0 && scale_last) ? 1 : 0;
    // the inverse pass keeps the CTA-wide kernel in auto mode: the warp-per-column inverse needs
    // two column slices per warp (3 CTAs/SM) and measured slower (batch 1024 x 2^18: 4.22 vs 3.89 ms)
    TcLayout tl;
    const bool tc = tc_layout_of(P, geom, npoly, lv, &tl);
    int kind = (P->pass_mode && !tc) ? pass_kind(P, cols) : 1;
    if (g.peer_mode && lv == lv_lo) {  // fused exchange: CTA kernel, stores to the owning ranks
      set_peer(A, g);
      kind = 1;
    }
    if (tc) {
      // table twiddles first (the last level with the pre-scaled rows), then the pass multiplies
      // only the untwiddled elements (scale mode 2) and runs the column DFT
      int rc;
      if ((rc = launch_tc_layout(P, poly, tl, A.scale != 0, s))) return rc;
      A.tw_skip = 1;
    }
    if (kind == 1 && A.scale) {
      // CTA-wide kernel: the twiddle products use the scaled rows, only untwiddled elements
      // take an explicit multiply (scale mode 2)
      A.scale = 2;
      A.twr = P->d_twr_s;
    }
    if (kind == 3) {
      PassArgs B = A;
      B.scale = 0;
      launch_tw(P, B, cols, s);
      CUCHK(cudaGetLastError());
      launch_dft(P, A, cols, s);
    } else if (kind == 2 && P->grid_iw) {
      A.wpc = 1;
      const int gw = (int)std::min<long long>(P->grid_iw, (cols + kWarpsPerCta - 1) / kWarpsPerCta);
      launch_k(P->kt.inv_w, dim3(gw), dim3(kWarpsPerCta * 32), P->kt.smem_inv_w, s, A, P->mc);
    } else if (A.tw_skip && P->grid_pass_do) {  // DFT only: three CTAs per SM
      const long long tiles = (cols + P->kt.cols_do - 1) / P->kt.cols_do;
      const int gd = (int)std::min<long long>(tiles, P->grid_pass_do);
      A.ctr = next_tick(P, tiles, gd);
      launch_k(P->kt.inv_do, dim3(gd), dim3(P->kt.nt), P->kt.smem_pass_do, s, A, P->mc);
    } else {
      A.ctr = next_tick(P, (cols + P->kt.cols - 1) / P->kt.cols, grid);
      launch_k(P->kt.inv, dim3(grid), dim3(P->kt.nt), smem_pass(P), s, A, P->mc);
    }
    CUCHK(cudaGetLastError());
    mark(P, s, DKSS_K_INV_PASS, tc ? 0 : (long long)(share * rp_work(P, npoly * level_twiddles(P, lv))),
         2LL * cols * 2 * P->m * P->m * P->L * 4);
  }
  return 0;
}

int launch_bottom(dkss_plan* P, uint32_t* a, const uint32_t* b, int npoly, int mode, bool scale, cudaStream_t s) {
  BottomArgs A{};
  A.a = a;
  A.b = b;
  A.poly_words = P->poly_words;
  A.elems_per_poly = 2LL * P->M;
  A.logb = P->logb;
  A.mode = mode;
  A.scale = scale ? 1 : 0;
  const long long elems = 2LL * P->M * npoly;
  const int grid = (int)std::min<long long>((elems + P->kt.ne - 1) / P->kt.ne, P->grid_bot);
  A.total_elems = elems;
  A.ctr = next_tick(P, (elems + P->kt.ne - 1) / P->kt.ne, grid);
  launch_k(P->kt.bottom, dim3(grid), dim3(P->kt.nt), smem_two(P), s, A, P->mc);
  CUCHK(cudaGetLastError());
  mark(P, s, DKSS_K_BOTTOM, mode ? rp_work(P, 2LL * P->M * npoly) : 0,
       (mode ? 3LL : 2LL) * npoly * P->poly_words * 4);
  return 0;
}

// carry resolution after a decode1-style kernel: one self-scanning kernel for products of at
// most kSelfScanBlocks blocks (DKSS_NO_SELFSCAN=1: always the scan + apply pair)
void launch_carry_tail(const DecodeArgs& A, int npoly, cudaStream_t s) {
  static const bool off = knob_on(DKSS_KNOB("DKSS_NO_SELFSCAN"));
  const dim3 grid((unsigned)(A.blocks_per_poly * npoly));
  if (!off && A.blocks_per_poly <= kSelfScanBlocks) {
    launch_k(k_decode2s, grid, dim3(kDecThreads), 0, s, A);
    return;
  }
  launch_k(k_decode_scan, dim3(npoly), dim3(kScanThreads), 0, s, A);
  launch_k(k_decode2, grid, dim3(kDecThreads), 0, s, A);
}

int launch_decode(dkss_plan* P, const uint32_t* v, uint32_t* out, int npoly, cudaStream_t s,
                  const unsigned long long* sglob = nullptr) {
  DecodeArgs A{};
  A.v = v;
  A.sglob = sglob;
  A.poly_words = P->poly_words;
  A.out = out;
  A.nout = P->prod_limbs;
  A.gmask = P->d_gmask;
  A.pmask = P->d_pmask;
  A.bstat = P->d_bstat;
  A.blocks_per_poly = dec_blocks(P);
  A.M = P->M;
  A.MM = P->m;
  A.L = P->L;
  A.u = P->u;
  const int grid = A.blocks_per_poly * npoly;
  void (*k1)(DecodeArgs) = k_decode1;
  if (!sglob && A.u == 32) {
    switch (A.L) {
      case 2: k1 = k_decode1_u32<2>; break;
      case 3: k1 = k_decode1_u32<3>; break;
      case 4: k1 = k_decode1_u32<4>; break;
      case 5: k1 = k_decode1_u32<5>; break;
      case 6: k1 = k_decode1_u32<6>; break;
      default: break;
    }
  }
  launch_k(k1, dim3(grid), dim3(kDecThreads), 0, s, A);
  CUCHK(cudaGetLastError());
  mark(P, s, DKSS_K_DECODE1, 0, npoly * (P->poly_words * 4 + P->prod_limbs * 4));
  launch_carry_tail(A, npoly, s);
  CUCHK(cudaGetLastError());
  mark(P, s, DKSS_K_DECODE2, 0, npoly * 2LL * P->prod_limbs * 4);
  return 0;
}

// row phase (levels 1.. of both transforms and the pointwise products) in one cluster kernel
int launch_rows(dkss_plan* P, uint32_t* a, const uint32_t* b, int batch, bool sq, cudaStream_t s) {
  RowsArgs R{};
  R.a = a;
  R.b = b;
  R.poly_words = P->poly_words;
  R.rows = (long long)batch * 2 * P->m;
  R.log_top_mu = P->log_top_mu;
  R.twr = P->d_twr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(R.rows * P->rows_cs));
  cfg.blockDim = dim3(P->kt.nt);
  cfg.dynamicSmemBytes = P->kt.smem_rows;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->rows_cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  CUCHK(cudaLaunchKernelEx(&cfg, P->rows_fn, R, P->mc));
  count_launch();
  const long long lt1 = level_twiddles(P, 1);
  mark(P, s, DKSS_K_ROWS, rp_work(P, (sq ? 2 : 3) * batch * lt1 + 2LL * P->M * batch),
       (sq ? 2LL : 3LL) * batch * P->poly_words * 4);
  return 0;
}

// row phase (levels 1.. of both transforms, pointwise, inverse levels 1..) as one persistent
// kernel with per-row dependency counters (dkss_dyn.cuh)
int launch_dyn(dkss_plan* P, uint32_t* a, const uint32_t* b, int batch, bool sq, cudaStream_t s, int rows_pp = 0) {
  const int E = rows_pp ? rows_pp : 2 * P->m;
  DynArgs R{};
  R.rows_pp = E;
  R.a = a;
  R.b = b;
  R.poly_words = P->poly_words;
  R.batch = batch;
  R.npolys_fwd = sq ? 1 : 2;
  R.log_mu0 = P->log_top_mu;
  R.log_mu1 = P->log_top_mu - P->logE;
  R.log_top_mu = P->log_top_mu;
  R.logb = P->logb;
  R.twr = P->d_twr;
  R.ticket = P->d_dyn;
  R.fwd_done = P->d_dyn + 4;
  R.bot_done = P->d_dyn + 4 + (size_t)batch * E;
  const unsigned rows = (unsigned)batch * E, mu1 = 1u << R.log_mu1;
  R.n_f = rows * R.npolys_fwd * mu1;
  R.n_b = rows * (unsigned)((1LL << R.log_mu0) / P->kt.ne);
  R.n_i = rows * mu1;
  R.rows = rows;  // counters start at zero (ensure_ws) and the kernel's last CTA re-zeroes them
  launch_k(P->kt.dyn, dim3(P->dyn_grid), dim3(P->kt.nt), P->kt.smem_dyn, s, R, P->mc);
  CUCHK(cudaGetLastError());
  const long long lt1 = level_twiddles(P, 1);
  mark(P, s, DKSS_K_ROWS, rp_work(P, (sq ? 2 : 3) * batch * lt1 + 2LL * P->M * batch),
       (sq ? 6LL : 9LL) * batch * P->poly_words * 4);
  return 0;
}

// whole multiply: operands already encoded-able in device memory
// b == nullptr: squaring (one forward transform; the pointwise step multiplies each
// transformed element by itself -- the reference's LL loop squares, bigmul/bench.py:214-215)
int run_mul(dkss_plan* P, int batch, const uint32_t* a, const uint32_t* b, long long nl, uint32_t* prod,
            cudaStream_t s) {
  const bool sq = b == nullptr;
  uint32_t* pa = P->d_poly;
  uint32_t* pb = sq ? pa : P->d_poly + (size_t)batch * P->poly_words;
  int rc;
  if (P->rows_cs || P->dyn_grid) {
    // level 0 (with the encode) over columns; everything inside a row in one kernel (cluster
    // or persistent dependency-driven); level 0 of the inverse with the 1/2M scale
    if ((rc = launch_fwd_levels(P, P->d_poly, (sq ? 1 : 2) * batch, s, a, b, nl, batch, 0, 1))) return rc;
    if ((rc = P->rows_cs ? launch_rows(P, pa, pb, batch, sq, s) : launch_dyn(P, pa, pb, batch, sq, s))) return rc;
    if ((rc = launch_inv_levels(P, pa, batch, true, s, 0, 1))) return rc;
    return launch_decode(P, pa, prod, batch, s);
  }
  if (P->levels > 0) {
    // encode fused into the first forward pass
    if ((rc = launch_fwd_levels(P, P->d_poly, (sq ? 1 : 2) * batch, s, a, b, nl, batch))) return rc;
  } else {
    if ((rc = launch_encode(P, a, nl, pa, batch, s))) return rc;
    if (!sq && (rc = launch_encode(P, b, nl, pb, batch, s))) return rc;
  }
#ifdef DKSS_EXPERIMENTS
  // DKSS_EXP_SKIP (timing experiments only, wrong products): bit 0 bottom, 1 inverse, 2 decode
  static const int skip = [] {
    const char* e = getenv("DKSS_EXP_SKIP");
    return e ? atoi(e) : 0;
  }();
#else
  constexpr int skip = 0;
#endif
  if (!(skip & 1) && (rc = launch_bottom(P, pa, pb, batch, 1, P->levels == 0, s))) return rc;
  if (!(skip & 2) && (rc = launch_inv_levels(P, pa, batch, true, s))) return rc;
  if (!(skip & 4) && (rc = launch_decode(P, pa, prod, batch, s))) return rc;
  return 0;
}

// One product in two parts (the host digits path, run_digits_split): part 0 is operand a's first
// transform level (fused encode + column DFT; its table twiddles wait for b), part 1 the same for
// b, then level 0's table twiddles of both polynomials in one launch and the rest of run_mul --
// or, for large operands, each operand's whole forward transform in its own part (below).
// Same kernels and products as run_mul.
bool split_ok(const dkss_plan* P) { return P->levels > 0 && !P->rows_cs && !P->dyn_grid; }

int run_mul_part(dkss_plan* P, int part, const uint32_t* op, long long nl, uint32_t* prod, cudaStream_t s) {
  uint32_t* pa = P->d_poly;
  uint32_t* pb = P->d_poly + P->poly_words;
  int rc;
  // From 2^23-bit operands on, each part runs its operand's WHOLE forward transform (single-
  // polynomial tensor-core launches): b's transfer (138 us at 2^24) is much longer than a's first
  // level (25 us), and the extra device time of the unbatched launches (~40 us at 2^24) is less
  // than the transfer it hides: dmul(int, int) 880 -> 845 us at 2^24, 3090 -> 2897 us at 2^26;
  // below that the batched forward wins (2^21: 227 vs 242 us, 2^22: 282 vs 285 us).
  const bool full_a = P->N >= (1LL << 23) && use_tc(P, 1);
  if (full_a) {
    if ((rc = launch_fwd_levels(P, part ? pb : pa, 1, s, op, nullptr, nl, 1))) return rc;
    if (part == 0) return 0;
    if ((rc = launch_bottom(P, pa, pb, 1, 1, false, s))) return rc;
    if ((rc = launch_inv_levels(P, pa, 1, true, s))) return rc;
    return launch_decode(P, pa, prod, 1, s);
  }
  if ((rc = launch_fwd_levels(P, part ? pb : pa, 1, s, op, nullptr, nl, 1, 0, 1, nullptr, 2, false))) return rc;
  if (part == 0) return 0;
  if (use_tc(P, 2) && (rc = launch_tc(P, pa, 2, 0, false, s))) return rc;
  if (P->levels > 1 && (rc = launch_fwd_levels(P, pa, 2, s, nullptr, nullptr, 0, 0, 1))) return rc;
  if ((rc = launch_bottom(P, pa, pb, 1, 1, false, s))) return rc;
  if ((rc = launch_inv_levels(P, pa, 1, true, s))) return rc;
  return launch_decode(P, pa, prod, 1, s);
}

int check_operand(const dkss_plan* P, const uint32_t* a, size_t na) {
  // value must be < 2^N (bigmul/dkss.py:389-390)
  for (size_t i = na; i-- > 0;) {
    if (!a[i]) continue;
    const long long top = 32LL * (long long)i + (31 - __builtin_clz(a[i]));
    if (top >= P->N) return fail(DKSS_ERANGE, "operand does not fit the plan (bit %lld >= N=%lld)", top, P->N);
    break;
  }
  return 0;
}

int plan_init(dkss_plan* P, const dkss_plan_desc* d, const dkss_plan_opts& opts, const KTable& kt, int device);

}  // namespace

// =====================================================================================
extern "C" {

int dkss_version(void) { return 1; }

int64_t dkss_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int64_t dkss_footprint_bytes(int64_t N, int32_t M, int32_t m, int32_t L) {
  if (N < 1 || M < m || m < 2 || L < 2) return -1;
  // what a batch-1 multiply through dkss_mul_digits holds on the device: plan_init's tables
  // (d_tw, d_twr, d_twr_s), ensure_ws(P, 1), the digits staging of run_digits_graph (30-bit digits)
  const long long op = (N + 31) / 32, prod = (2 * N + 31) / 32, poly_b = 2LL * M * m * L * 4;
  const long long blocks = (prod + kDecThreads - 1) / kDecThreads;
  const long long tables = (long long)(M / m) * m * L * 4 * (1 + 2 + 2);
  const long long ws = 2 * poly_b + 2 * op * 4 + prod * 4 + blocks * kDecWarps * 8 + blocks * 4 +
                       (4 + 2LL * 2 * m) * 4 + 2LL * kTickSlots * 4;
  const long long stage = 4 * (2 * 3 + 2 * ((N + 29) / 30));
  return tables + ws + stage;
}

const char* dkss_last_error(void) { return g_err.c_str(); }

int dkss_plan_create(const dkss_plan_desc* d, int device, dkss_plan** out) {
  return dkss_plan_create_ex(d, nullptr, device, out);
}

int dkss_plan_create_ex(const dkss_plan_desc* d, const dkss_plan_opts* o, int device, dkss_plan** out) {
  const dkss_plan_opts opts = o ? *o : dkss_plan_opts{};
  if (!d || !out || !d->p || !d->rho_powers) return fail(DKSS_EINVAL, "null argument");
  *out = nullptr;
  const int M = d->M, m = d->m, L = d->L;
  if (M < m || m < 2 || (M & (M - 1)) || (m & (m - 1))) return fail(DKSS_EINVAL, "M and m must be powers of 2, M >= m");
  if (L < 2 || L > DKSS_MAXL) return fail(DKSS_EINVAL, "L=%d unsupported (2..%d)", L, DKSS_MAXL);
  if (d->p[L - 1] == 0 || !(d->p[0] & 1)) return fail(DKSS_EINVAL, "p must be odd with exactly L=%d limbs", L);
  KTable kt;
  if (!lookup(m, L, &kt)) return fail(DKSS_EINVAL, "no kernels for m=%d, L=%d (m in {8,16,32})", m, L);
  if (opts.row_phase < DKSS_ROWS_AUTO || opts.row_phase > DKSS_ROWS_CLUSTER || opts.pass_kind < DKSS_PASS_AUTO ||
      opts.pass_kind > DKSS_PASS_SPLIT || opts.twiddle < DKSS_TWIDDLE_AUTO || opts.twiddle > DKSS_TWIDDLE_TENSOR)
    return fail(DKSS_EINVAL, "bad plan options (row_phase %d, pass_kind %d, twiddle %d)", opts.row_phase,
                opts.pass_kind, opts.twiddle);
  CUCHK(cudaSetDevice(device));
  dkss_plan* P = new dkss_plan();
  const int rc = plan_init(P, d, opts, kt, device);
  if (rc) {
    dkss_plan_destroy(P);  // every partially built resource is released on the error paths
    return rc;
  }
  *out = P;
  return DKSS_OK;
}

}  // extern "C"

namespace {
int plan_init(dkss_plan* P, const dkss_plan_desc* d, const dkss_plan_opts& opts, const KTable& kt, int device) {
  const int M = d->M, m = d->m, L = d->L;
  P->device = device;
  P->N = d->N;
  P->M = M;
  P->m = m;
  P->u = d->u;
  P->L = L;
  P->kt = kt;
  P->logE = ilog2i(2 * m);
  const int logn = ilog2i(2LL * M);
  P->levels = 0;
  long long n = 2LL * M;
  while (n > 2 * m) {
    n /= 2 * m;
    P->levels++;
  }
  P->base_len = (int)n;
  P->logb = ilog2i(n);
  P->log_top_mu = ilog2i((long long)M / m);
  (void)logn;
  P->poly_words = 2LL * M * m * L;
  P->op_limbs = (d->N + 31) / 32;
  P->prod_limbs = (2 * d->N + 31) / 32;
  {
    long long tw = 0, len = 2LL * M, inst = 1;
    while (len > 2 * m) {
      const long long mu = len / (2 * m);
      tw += inst * (2 * m - 1) * (mu - 1);
      inst *= 2 * m;
      len = mu;
    }
    P->twiddles = tw;
  }
  // modulus constants
  Limbs p(d->p, d->p + L);
  memcpy(P->mc.p, d->p, 4 * L);
  uint32_t inv = 1;
  for (int i = 0; i < 5; ++i) inv *= 2u - p[0] * inv;
  P->mc.pinv = 0u - inv;
  {
    bool pr = L >= 2 && p[0] == 1u;
    for (int i = 1; i + 1 < L; ++i) pr = pr && p[i] == 0u;
    P->mc.proth = (pr && !knob_on(DKSS_KNOB("DKSS_NO_PROTH"))) ? 1u : 0u;
  }
  {
    // qbias = p * 2^(32L + 5) in 2L+1 limbs (pointwise bias removal, ring_mul BiasFromY)
    uint64_t carry = 0;
    for (int i = 0; i < 2 * L + 1; ++i) P->mc.qbias[i] = 0;
    for (int i = 0; i < L; ++i) {
      const uint64_t v = ((uint64_t)p[i] << 5) | carry;
      P->mc.qbias[L + i] = (uint32_t)v;
      carry = v >> 32;
    }
    P->mc.qbias[2 * L] = (uint32_t)carry;
  }
  Limbs x(L, 0);
  x[0] = 1;
  for (int i = 0; i < 32 * L; ++i) dbl_mod(x, p);
  Limbs rmod = x;  // R mod p
  for (int i = 0; i < 32 * L; ++i) dbl_mod(x, p);
  memcpy(P->mc.r2, x.data(), 4 * L);  // R^2 mod p
  Limbs ks = x;
  for (int i = 0; i < logn; ++i) half_mod(ks, p);
  memcpy(P->mc.kscale, ks.data(), 4 * L);
  Limbs ki = rmod;
  for (int i = 0; i < logn; ++i) half_mod(ki, p);
  memcpy(P->mc.kinv, ki.data(), 4 * L);
  double pd = 0;
  for (int i = L - 1; i >= 0; --i) pd = pd * 4294967296.0 + p[i];
  P->mc.pf_inv = (float)(ldexp(1.0, 32 * (L - 2)) / pd);
  // kernels: opt into >48 KB dynamic smem
  // kernels: opt into >48 KB dynamic smem and the max-shared carveout; persistent grids
  {
    const void* fns[4] = {(const void*)kt.fwd, (const void*)kt.inv, (const void*)kt.bottom, (const void*)kt.rmul};
    const size_t need[4] = {kt.smem_pass, kt.smem_pass, kt.smem_bot, kt.smem_rmul};
    for (int i = 0; i < 4; ++i) {
      CUCHK(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need[i]));
      CUCHK(cudaFuncSetAttribute(fns[i], cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    int sms = 0, occ_f = 0, occ_i = 0, occ_b = 0;
    CUCHK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, kt.fwd, kt.nt, kt.smem_pass));
    CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_i, kt.inv, kt.nt, kt.smem_pass));
    CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, kt.bottom, kt.nt, kt.smem_bot));
    if (occ_f < 1 || occ_i < 1 || occ_b < 1) return fail(DKSS_EINVAL, "kernels for m=%d L=%d do not fit an SM", m, L);
    P->grid_pass = sms * std::min(occ_f, occ_i);
    P->grid_bot = sms * occ_b;
    if (kt.fwd_do && !knob_on(DKSS_KNOB("DKSS_NO_DFT_ONLY"))) {
      int od_f = 0, od_i = 0;
      for (const void* f : {(const void*)kt.fwd_do, (const void*)kt.inv_do}) {
        CUCHK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_pass_do));
        CUCHK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      }
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od_f, kt.fwd_do, kt.nt, kt.smem_pass_do));
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od_i, kt.inv_do, kt.nt, kt.smem_pass_do));
      P->grid_pass_do = sms * std::min(od_f, od_i);
    }
    if (kt.fwd_w && !knob_on(DKSS_KNOB("DKSS_NO_WARP_PASS"))) {
      int ofw = 0, oiw = 0;
      CUCHK(cudaFuncSetAttribute((const void*)kt.fwd_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_fwd_w));
      CUCHK(cudaFuncSetAttribute((const void*)kt.inv_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_inv_w));
      CUCHK(cudaFuncSetAttribute((const void*)kt.fwd_w, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      CUCHK(cudaFuncSetAttribute((const void*)kt.inv_w, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ofw, kt.fwd_w, kWarpsPerCta * 32, kt.smem_fwd_w));
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oiw, kt.inv_w, kWarpsPerCta * 32, kt.smem_inv_w));
      P->grid_fw = ofw > 0 ? sms * ofw : 0;
      P->grid_iw = oiw > 0 ? sms * oiw : 0;
    }
    if (kt.dft) {
      int od = 0;
      CUCHK(cudaFuncSetAttribute((const void*)kt.dft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_dft));
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od, kt.dft, kWarpsPerCta * 32, kt.smem_dft));
      P->grid_dft = od > 0 ? sms * od : 0;
    }
    {
      int ot = 0;
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ot, kt.tw, 256, 0));
      P->grid_tw = sms * std::max(ot, 1);
    }
    P->pass_mode = opts.pass_kind;
    // table twiddles on the tensor cores: kernels exist for m in {16, 32} at L = 4, the epilogue
    // needs a Proth prime p = 1 + p3 2^96, and the split column passes are CTA kernels
    {
      // epilogue bounds (dkss_tc.cuh reduce_coeff16): p in (2^127, 2^128 - 2^113), and p / 2 within
      // the range of 16 balanced base-256 digits
      const bool tc_ok = kt.tc && L == 4 && P->mc.proth && P->levels >= 1 && d->p[1] == 0 && d->p[2] == 0 &&
                         d->p[3] >= 0x80000000u && d->p[3] <= 0xFEFEFEFEu;
      if (opts.twiddle == DKSS_TWIDDLE_TENSOR && !tc_ok)
        return fail(DKSS_EINVAL, "tensor-core twiddles need m in {16, 32}, L = 4 and a Proth prime (m=%d L=%d)", m, L);
      P->tc = tc_ok && opts.twiddle != DKSS_TWIDDLE_CUDA && P->pass_mode <= DKSS_PASS_CTA;
      P->tc_forced = P->tc && opts.twiddle == DKSS_TWIDDLE_TENSOR;
      if (P->tc) {
        P->tc_p3 = d->p[3];
        P->tc_grid = sms;
        CUCHK(cudaFuncSetAttribute((const void*)kt.tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_tc));
      }
    }
    // row phase in one cluster kernel: two column levels, base length b = cluster size.
    // Opt-in (DKSS_ROWS_CLUSTER): measured slower than the three persistent launches it replaces
    // -- second-level column 0 has no twiddles, so one CTA of every
    // cluster idles through both level-1 phases, and the cluster barriers keep the CTAs in
    // lockstep where the persistent kernels overlap tiles
    const int b = P->base_len;
    const int ri = b == 2 ? 1 : b == 4 ? 2 : b == 8 ? 3 : b == 16 ? 4 : 0;
    if (!P->tc && P->levels == 2 && ri && kt.rows[ri] && opts.row_phase == DKSS_ROWS_CLUSTER) {
      auto fn = kt.rows[ri];
      bool ok = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_rows) ==
                cudaSuccess;
      if (ok && b > 8)
        ok = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
      if (ok) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(b * 2 * m);
        cfg.blockDim = dim3(kt.nt);
        cfg.dynamicSmemBytes = kt.smem_rows;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = b;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        ok = cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) == cudaSuccess && ncl > 0;
      }
      cudaGetLastError();  // a refused configuration keeps the three-launch row phase
      if (ok) {
        P->rows_cs = b;
        P->rows_fn = fn;
      }
    }
    // row phase as one persistent dependency-driven kernel: default for m = 32 two-level plans
    // with a base case of 4 to 16 (2^24: 1.375 vs 1.389 ms; 2^22: 434 vs 443 us); at 2^26
    // (b = 64), at 2^21 (b = 2: 289 vs 267 us) and for m = 16 the three ticketed launches
    // measured faster.  DKSS_ROWS_PERSISTENT forces it on, DKSS_ROWS_LAUNCHES off.
    const bool want_dyn = opts.row_phase == DKSS_ROWS_PERSISTENT ||
                          (opts.row_phase == DKSS_ROWS_AUTO && m == 32 && P->base_len >= 4 && P->base_len <= 16);
    if (!P->tc && !P->rows_cs && P->levels == 2 && kt.dyn && want_dyn &&
        (1LL << P->log_top_mu) % kt.ne == 0) {
      CUCHK(cudaFuncSetAttribute((const void*)kt.dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kt.smem_dyn));
      int od = 0;
      CUCHK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&od, kt.dyn, kt.nt, kt.smem_dyn));
      P->dyn_grid = od > 0 ? sms * od : 0;
    }
  }
  // cbias = -(2^(32L) - 1) * R mod p = (p - ((R mod p) - 1)) * R mod p  (ring_mul bias correction)
  {
    Limbs b = rmod;  // R mod p
    // b = (R mod p) - 1  (R mod p != 0 since p is odd and > 1)
    for (int i = 0; i < L; ++i) {
      if (b[i]--) break;
    }
    Limbs nb(L, 0);  // p - b  (b in [0, p))
    bool bz = true;
    for (int i = 0; i < L; ++i) bz = bz && b[i] == 0;
    if (!bz) {
      nb = p;
      sub_inplace(nb, b);
    }
    for (int i = 0; i < 32 * L; ++i) dbl_mod(nb, p);  // * R
    memcpy(P->mc.cbias, nb.data(), 4 * L);
  }
  CUCHK(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
  {
    P->dyn_tiles = !knob_on(DKSS_KNOB("DKSS_NO_DYNTILES"));
    CUCHK(cudaMalloc(&P->d_tick, 2 * kTickSlots * sizeof(unsigned)));
    CUCHK(upload_sync(P->d_tick, nullptr, 2 * kTickSlots * sizeof(unsigned)));
  }
  // twiddle table -> Montgomery form
  const size_t tw_words = (size_t)(M / m) * m * L;
  cudaError_t e = cudaMalloc(&P->d_tw, tw_words * 4);
  if (e == cudaSuccess) e = upload_sync(P->d_tw, d->rho_powers, tw_words * 4);
  if (e == cudaSuccess) {
    count_launch();
    kt.mscale<<<(int)std::min<size_t>((tw_words / L + 255) / 256, 4096), 256, 0, P->stream>>>(P->d_tw, tw_words / L, 0,
                                                                                               P->mc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMalloc(&P->d_twr, (size_t)(M / m) * 2 * m * L * 4);
  if (e == cudaSuccess) {
    count_launch();
    kt.build_twr<<<(int)std::min<size_t>(((size_t)(M / m) * m + 255) / 256, 4096), 256, 0, P->stream>>>(
        P->d_tw, P->d_twr, (long long)(M / m), m, P->mc);
    e = cudaGetLastError();
  }
  // scaled rows for the last inverse level: rho^s R * kscale R^-1 = rho^s (2M)^-1 R^2, so a
  // twiddle product also applies the final 1/2M (and undoes the pointwise R^-1)
  uint32_t* tw_s = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&tw_s, tw_words * 4);
  if (e == cudaSuccess) e = cudaMemcpyAsync(tw_s, P->d_tw, tw_words * 4, cudaMemcpyDeviceToDevice, P->stream);
  if (e == cudaSuccess) {
    count_launch();
    kt.mscale<<<(int)std::min<size_t>((tw_words / L + 255) / 256, 4096), 256, 0, P->stream>>>(tw_s, tw_words / L, 2,
                                                                                               P->mc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMalloc(&P->d_twr_s, (size_t)(M / m) * 2 * m * L * 4);
  if (e == cudaSuccess) {
    count_launch();
    kt.build_twr<<<(int)std::min<size_t>(((size_t)(M / m) * m + 255) / 256, 4096), 256, 0, P->stream>>>(
        tw_s, P->d_twr_s, (long long)(M / m), m, P->mc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && P->tc) {
    // V tables of the tensor-core twiddles, from the expanded rows; ck[k] = 2^(32 + 8k) mod p
    std::vector<uint32_t> ck;
    {
      Limbs c(L, 0);
      c[0] = 1;
      for (int i = 0; i < 32; ++i) dbl_mod(c, p);
      for (int k = 0; k < 16; ++k) {
        ck.insert(ck.end(), c.begin(), c.end());
        for (int i = 0; i < 8; ++i) dbl_mod(c, p);
      }
    }
    uint32_t* d_c = nullptr;
    const size_t vbytes = (size_t)(M / m) * kt.tc_vbytes;
    e = cudaMalloc(&d_c, 4 * ck.size());
    if (e == cudaSuccess) e = upload_sync(d_c, ck.data(), 4 * ck.size());
    if (e == cudaSuccess) e = cudaMalloc(&P->d_vtab, vbytes);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_vtab_s, vbytes);
    const int gb = (int)std::min<long long>(((long long)(M / m) * (2 * m - 1) + 127) / 128, 4096);
    if (e == cudaSuccess) {
      count_launch();
      kt.tc_build<<<gb, 128, 0, P->stream>>>(P->d_twr, (long long)(M / m), P->d_vtab, P->mc, d_c);
      count_launch();
      kt.tc_build<<<gb, 128, 0, P->stream>>>(P->d_twr_s, (long long)(M / m), P->d_vtab_s, P->mc, d_c);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
    cudaFree(d_c);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
  cudaFree(tw_s);
  if (e != cudaSuccess) return fail(DKSS_ECUDA, "plan upload failed: %s", cudaGetErrorString(e));
  return 0;
}
}  // namespace

extern "C" {

void dkss_plan_destroy(dkss_plan* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  free_ws(P);
  cudaFree(P->d_tw);
  cudaFree(P->d_twr);
  cudaFree(P->d_twr_s);
  cudaFree(P->d_tick);
  cudaFree(P->d_vtab);
  cudaFree(P->d_vtab_s);
  for (auto& kv : P->tc_sched) {
    cudaFree(kv.second.d_tiles);
    cudaFree(kv.second.d_entries);
  }
  if (P->h_pin) cudaFreeHost(P->h_pin);
  cudaFree(P->d_stage);
  cudaFree(P->d_sglob);
  if (P->stream) cudaStreamDestroy(P->stream);
  if (P->cstream) cudaStreamDestroy(P->cstream);
  for (cudaEvent_t e : P->ev_ops)
    if (e) cudaEventDestroy(e);
  delete P;
}

int dkss_plan_get_info(const dkss_plan* P, dkss_plan_info* o) {
  if (!P || !o) return fail(DKSS_EINVAL, "null argument");
  o->N = P->N;
  o->M = P->M;
  o->m = P->m;
  o->u = P->u;
  o->L = P->L;
  o->levels = P->levels;
  o->base_len = P->base_len;
  o->poly_bytes = P->poly_words * 4;
  o->operand_limbs = P->op_limbs;
  o->product_limbs = P->prod_limbs;
  o->twiddles_per_fft = P->twiddles;
  o->ring_products = 3 * P->twiddles + 2LL * P->M;
  {
    const bool self = !knob_on(DKSS_KNOB("DKSS_NO_SELFSCAN")) && dec_blocks(P) <= kSelfScanBlocks;
    const int dec = self ? 2 : 3;  // decode1 + (self-scanning apply | scan + apply)
    o->launches_per_mul =
        (P->rows_cs || P->dyn_grid) ? 1 + 1 + 1 + dec
                                    : (P->levels > 0 ? 0 : 2) + P->levels * (use_tc(P, 2) ? 2 : 1) * 2 + 1 + dec;
  }
  o->workspace_bytes = (int64_t)P->ws_bytes;
  o->footprint_bytes = dkss_footprint_bytes(P->N, P->M, P->m, P->L);
  return DKSS_OK;
}

}  // extern "C"

namespace {
// capture (once) and replay the whole multiply for fixed (pointers, batch, sizes)
int launch_graph(dkss_plan* P, int batch, const uint32_t* a, const uint32_t* b, size_t nl, uint32_t* c, size_t nc,
                 cudaStream_t s) {
  int rc;
  if ((rc = ensure_ws(P, batch))) return rc;
  GraphKey key{batch, a, b, c, nl, nc};
  auto* ent = P->graphs.find(key);
  if (!ent) {
    if ((rc = tc_prepare(P, batch, b == nullptr))) return rc;
    cudaStream_t cap;
    CUCHK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CUCHK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    {
      CaptureScope cs;
      rc = run_mul(P, batch, a, b, (long long)nl, P->d_prod, cap);
    }
    if (!rc && c != P->d_prod) {
      if ((long long)nc == P->prod_limbs) {
        cudaMemcpyAsync(c, P->d_prod, (size_t)batch * P->prod_limbs * 4, cudaMemcpyDeviceToDevice, cap);
      } else {
        cudaMemsetAsync(c, 0, (size_t)batch * nc * 4, cap);
        cudaMemcpy2DAsync(c, nc * 4, P->d_prod, P->prod_limbs * 4, P->prod_limbs * 4, batch,
                          cudaMemcpyDeviceToDevice, cap);
      }
    }
    cudaGraph_t g;
    cudaError_t e = cudaStreamEndCapture(cap, &g);
    cudaStreamDestroy(cap);
    if (rc) {
      if (e == cudaSuccess) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(DKSS_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    if (!(ent = P->graphs.put(key, g, &e))) return fail(DKSS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  }
  CUCHK(P->graphs.launch(ent, s));
  return 0;
}
}  // namespace

extern "C" {

int dkss_mul_device(dkss_plan* P, int batch, const uint32_t* a, const uint32_t* b, size_t nl, uint32_t* c, size_t nc,
                    void* stream) {
  if (!P || batch < 1 || !a || !c) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nl > P->op_limbs) return fail(DKSS_ERANGE, "operand limbs %zu exceed plan (%lld)", nl, P->op_limbs);
  if ((long long)nc < P->prod_limbs) return fail(DKSS_EINVAL, "nc=%zu below product limbs %lld", nc, P->prod_limbs);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  return launch_graph(P, batch, a, b, nl, c, nc, (cudaStream_t)stream);
}

int dkss_profile_device(dkss_plan* P, int batch, const uint32_t* a, const uint32_t* b, size_t nl, uint32_t* c,
                        void* stream, int max_launches, int32_t* kinds, float* ms, int64_t* work, int64_t* bytes,
                        int* n_launches) {
  if (!P || batch < 1 || !a || !b || !c || !kinds || !ms || !n_launches) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nl > P->op_limbs) return fail(DKSS_ERANGE, "operand limbs exceed plan");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, batch))) return rc;
  dkss_plan::Prof pr;
  for (int i = 0; i <= dkss_plan::Prof::kMax; ++i) CUCHK(cudaEventCreate(&pr.ev[i]));
  cudaStream_t s = (cudaStream_t)stream;
  P->prof = &pr;
  cudaEventRecord(pr.ev[0], s);
  rc = run_mul(P, batch, a, b, (long long)nl, c, s);
  P->prof = nullptr;
  cudaError_t e = cudaStreamSynchronize(s);
  if (!rc && e != cudaSuccess) rc = fail(DKSS_ECUDA, "profile run failed: %s", cudaGetErrorString(e));
  if (!rc) {
    const int n = std::min(pr.n, max_launches);
    for (int i = 0; i < n; ++i) {
      kinds[i] = pr.kind[i];
      cudaEventElapsedTime(&ms[i], pr.ev[i], pr.ev[i + 1]);
      if (work) work[i] = pr.work[i];
      if (bytes) bytes[i] = pr.bytes[i];
    }
    *n_launches = n;
  }
  for (int i = 0; i <= dkss_plan::Prof::kMax; ++i) cudaEventDestroy(pr.ev[i]);
  return rc;
}

int dkss_mul_batch(dkss_plan* P, int batch, const uint32_t* a, const uint32_t* b, size_t nl, uint32_t* c, size_t nc) {
  if (!P || batch < 1 || !a || !b || !c) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nl > P->op_limbs) return fail(DKSS_ERANGE, "operand limbs %zu exceed plan (%lld)", nl, P->op_limbs);
  int rc;
  for (int i = 0; i < batch; ++i) {
    if ((rc = check_operand(P, a + (size_t)i * nl, nl))) return rc;
    if ((rc = check_operand(P, b + (size_t)i * nl, nl))) return rc;
  }
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  if ((rc = ensure_ws(P, batch))) return rc;
  const size_t opw = (size_t)batch * nl;
  const size_t prw = (size_t)batch * P->prod_limbs;
  if ((rc = ensure_pin(P, std::max(2 * opw, prw)))) return rc;
  cudaStream_t s = P->stream;
  memcpy(P->h_pin, a, opw * 4);
  memcpy(P->h_pin + opw, b, opw * 4);
  CUCHK(cudaMemcpyAsync(P->d_ops, P->h_pin, 2 * opw * 4, cudaMemcpyHostToDevice, s));
  if ((rc = launch_graph(P, batch, P->d_ops, P->d_ops + opw, nl, P->d_prod, P->prod_limbs, s))) return rc;
  CUCHK(cudaMemcpyAsync(P->h_pin, P->d_prod, prw * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  for (int i = 0; i < batch; ++i) {
    const uint32_t* src = P->h_pin + (size_t)i * P->prod_limbs;
    uint32_t* dst = c + (size_t)i * nc;
    const size_t ncopy = std::min<size_t>(nc, P->prod_limbs);
    memcpy(dst, src, ncopy * 4);
    for (size_t k = ncopy; k < (size_t)P->prod_limbs; ++k)
      if (src[k]) return fail(DKSS_ERANGE, "product does not fit nc=%zu limbs", nc);
    if (nc > ncopy) memset(dst + ncopy, 0, (nc - ncopy) * 4);
  }
  return DKSS_OK;
}

}  // extern "C"

namespace {
// DKSS_HOST_TIMING=1: host-side phase times of the host-buffer multiply, to stderr
struct HostTimer {
  bool on;
  std::chrono::steady_clock::time_point t0, last;
  char buf[512];
  int n = 0;
  HostTimer() {
    on = knob_on(DKSS_KNOB("DKSS_HOST_TIMING"));
    t0 = last = std::chrono::steady_clock::now();
    buf[0] = 0;
  }
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    n += snprintf(buf + n, sizeof buf - n, " %s=%.1f", what,
                  std::chrono::duration<double, std::micro>(now - last).count());
    last = now;
  }
  ~HostTimer() {
    if (on)
      fprintf(stderr, "dkss host us:%s total=%.1f\n", buf,
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
};
thread_local HostTimer* g_ht = nullptr;
void ht_mark(const char* w) {
  if (g_ht) g_ht->mark(w);
}

// Persistent host worker threads for the staging copies of the host-buffer entry points: a
// 4 MB operand copy is ~0.4 ms on one core; spread over the pool it overlaps the memory
// bandwidth of several cores (thread start-up per call would cost more than it saves).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* pool = new HostPool();  // never destroyed: workers outlive static teardown
    return *pool;
  }
  unsigned size() const { return (unsigned)workers_.size() + 1; }
  // fn(i) for i in [0, n) on the pool and the calling thread; returns when all are done
  void run(size_t n, const std::function<void(size_t)>& fn) {
    if (n == 0) return;
    if (n == 1 || workers_.empty()) {
      for (size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == n_; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = std::min(8u, hw) - 1;
    for (unsigned t = 0; t < nt; ++t)
      workers_.emplace_back([this] {
        unsigned long long seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
          }
          work();
        }
      });
    for (auto& w : workers_) w.detach();
  }
  void work() {
    for (;;) {
      size_t i;
      const std::function<void(size_t)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= n_) return;
        i = next_++;
        f = fn_;
      }
      (*f)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t n_ = 0, next_ = 0, done_ = 0;
  unsigned long long gen_ = 0;
};

constexpr size_t kCopyChunk = 512 << 10;  // bytes per staging-copy task

// memcpy in chunks over the host pool (small copies stay on the calling thread)
void par_memcpy(void* dst, const void* src, size_t bytes) {
  if (bytes < 2 * kCopyChunk) {
    if (bytes) memcpy(dst, src, bytes);
    return;
  }
  const size_t n = (bytes + kCopyChunk - 1) / kCopyChunk;
  HostPool::get().run(n, [&](size_t i) {
    const size_t off = i * kCopyChunk;
    memcpy((char*)dst + off, (const char*)src + off, std::min(kCopyChunk, bytes - off));
  });
}

// fn(i) for i in [0, n) over the host pool when `bytes` of copying is large
template <class F>
void host_par(size_t n, size_t bytes, F fn) {
  if (bytes < 2 * kCopyChunk || n <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  HostPool::get().run(n, [&](size_t i) { fn(i); });
}

bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// pinned host blocks handed out by dkss_host_alloc, recycled by size
struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_;  // size -> block
  std::map<void*, size_t> live;        // block -> size
  size_t cached = 0;
  static constexpr size_t kCacheCap = 512ull << 20;
};
PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool();
  return *p;
}

}  // namespace

namespace {
// Host digit strings -> products: the staging buffer (offsets + digits) goes to the device
// operand by operand as the host pool stages it, then ONE graph launch (radix repack, the
// multiply), then the D2H of the products -- straight into the caller's buffer when that is
// page-locked (dkss_host_alloc), else through the staging buffer.
// One product from host digits with the transfers overlapped: operand a is staged and sent
// (transfer stream), part 0 (a's repack + first transform level) starts as soon as it lands, b is
// staged on the host and sent while part 0 runs, then part 1 (b's repack + first level, the rest of
// the multiply).  The staging buffer holds the offsets header and a's then b's digits as in
// run_digits_graph.
int run_digits_split(dkss_plan* P, const std::vector<size_t>& nd, const uint32_t* const* ptrs, int digit_bits,
                     size_t head) {
  int rc;
  if (!P->cstream) {
    CUCHK(cudaStreamCreateWithFlags(&P->cstream, cudaStreamNonBlocking));
    CUCHK(cudaEventCreateWithFlags(&P->ev_ops[0], cudaEventDisableTiming));
    CUCHK(cudaEventCreateWithFlags(&P->ev_ops[1], cudaEventDisableTiming));
  }
  auto key_of = [&](int part) { return std::make_tuple(1, false, digit_bits | ((part + 1) << 8)); };
  for (int part = 0; part < 2; ++part) {
    if (P->dgraphs.find(key_of(part))) continue;
    if ((rc = tc_prepare(P, 1, false))) return rc;
    cudaStream_t cap_s;
    CUCHK(cudaStreamCreateWithFlags(&cap_s, cudaStreamNonBlocking));
    CUCHK(cudaStreamBeginCapture(cap_s, cudaStreamCaptureModeThreadLocal));
    {
      CaptureScope cs;
      RepackArgs R{};
      R.stage = P->d_stage + head;
      R.off = reinterpret_cast<const long long*>(P->d_stage) + part;
      R.dst = P->d_ops + (size_t)part * P->op_limbs;
      R.ndst = P->op_limbs;
      R.sbits = digit_bits;
      const int gx = (int)std::max<long long>(1, std::min<long long>((P->op_limbs + 255) / 256, 1184));
      launch_k(k_repack_bits, dim3(gx, 1), dim3(256), 0, cap_s, R);
      rc = run_mul_part(P, part, R.dst, P->op_limbs, P->d_prod, cap_s);
    }
    cudaGraph_t g;
    cudaError_t e = cudaStreamEndCapture(cap_s, &g);
    cudaStreamDestroy(cap_s);
    if (rc) {
      if (e == cudaSuccess) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(DKSS_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    if (!P->dgraphs.put(key_of(part), g, &e)) return fail(DKSS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  }
  auto* g0 = P->dgraphs.find(key_of(0));
  auto* g1 = P->dgraphs.find(key_of(1));
  if (!g0 || !g1) return fail(DKSS_ECUDA, "split graphs evicted");
  long long* off = reinterpret_cast<long long*>(P->h_pin);
  off[0] = 0;
  off[1] = (long long)nd[0];
  off[2] = (long long)(nd[0] + nd[1]);
  // the operands go to the device straight from the caller's (pageable) digits: the driver's
  // pageable path pipelines its own staging with the DMA -- 138 us for a 2^24-bit operand against
  // 216 us for a copy into our page-locked buffer followed by the transfer (tools/hostreg_probe.py).
  // Each pageable copy returns once staged, so b's transfer runs while part 0 computes.  (Issuing
  // the two from two host threads on two streams serialises them in the driver: 130 + 250 us.)
  // timing study (experiment builds, DKSS_HOST_TIMING=1): device-side events of the pieces
  const bool tev = g_ht && g_ht->on;
  cudaEvent_t te[6] = {};
  if (tev)
    for (auto& e : te) cudaEventCreate(&e);
  if (tev) cudaEventRecord(te[0], P->cstream);
  CUCHK(cudaMemcpyAsync(P->d_stage, P->h_pin, head * 4, cudaMemcpyHostToDevice, P->cstream));
  if (nd[0]) CUCHK(cudaMemcpyAsync(P->d_stage + head, ptrs[0], nd[0] * 4, cudaMemcpyHostToDevice, P->cstream));
  CUCHK(cudaEventRecord(P->ev_ops[0], P->cstream));
  if (tev) cudaEventRecord(te[1], P->cstream);
  CUCHK(cudaStreamWaitEvent(P->stream, P->ev_ops[0], 0));
  CUCHK(P->dgraphs.launch(g0, P->stream));
  if (tev) cudaEventRecord(te[2], P->stream);
  ht_mark("stage_launch_a");
  if (tev) cudaEventRecord(te[3], P->cstream);
  if (nd[1]) CUCHK(cudaMemcpyAsync(P->d_stage + head + nd[0], ptrs[1], nd[1] * 4, cudaMemcpyHostToDevice, P->cstream));
  CUCHK(cudaEventRecord(P->ev_ops[1], P->cstream));
  if (tev) cudaEventRecord(te[4], P->cstream);
  CUCHK(cudaStreamWaitEvent(P->stream, P->ev_ops[1], 0));
  CUCHK(P->dgraphs.launch(g1, P->stream));
  if (tev) cudaEventRecord(te[5], P->stream);
  ht_mark("stage_launch_b");
  if (tev) {
    cudaStreamSynchronize(P->stream);
    float t[5] = {};
    cudaEventElapsedTime(&t[0], te[0], te[1]);  // H2D a
    cudaEventElapsedTime(&t[1], te[1], te[2]);  // a landed -> part 0 done
    cudaEventElapsedTime(&t[2], te[3], te[4]);  // H2D b
    cudaEventElapsedTime(&t[3], te[4], te[5]);  // b landed -> part 1 done
    cudaEventElapsedTime(&t[4], te[0], te[5]);  // all
    fprintf(stderr, "dkss split dev us: h2d_a=%.1f part0=%.1f h2d_b=%.1f part1=%.1f first_h2d_to_end=%.1f\n",
            1e3 * t[0], 1e3 * t[1], 1e3 * t[2], 1e3 * t[3], 1e3 * t[4]);
    for (auto& e : te) cudaEventDestroy(e);
  }
  return 0;
}

int run_digits_graph(dkss_plan* P, int batch, bool sq, int nops, const uint32_t* const* ptrs, const size_t* counts,
                     int digit_bits, bool trusted, uint32_t* c, size_t nc) {
  std::vector<size_t> nd((size_t)nops);
  for (int q = 0; q < nops; ++q) {
    const uint32_t* d = ptrs[q];
    size_t n = counts[q];
    if (n && !d) return fail(DKSS_EINVAL, "null digit pointer");
    while (n > 0 && d[n - 1] == 0) --n;
    if (digit_bits < 32 && !trusted) {
      uint32_t any = 0;
      for (size_t i = 0; i < n; ++i) any |= d[i];
      if (any >> digit_bits) return fail(DKSS_EINVAL, "a digit exceeds %d bits", digit_bits);
    }
    if (n) {  // value < 2^N (bigmul/dkss.py:389-390)
      const uint32_t top = d[n - 1];
      if (digit_bits < 32 && (top >> digit_bits)) return fail(DKSS_EINVAL, "a digit exceeds %d bits", digit_bits);
      const long long bits = (long long)(n - 1) * digit_bits + (32 - __builtin_clz(top));
      if (bits > P->N) return fail(DKSS_ERANGE, "operand does not fit the plan (%lld bits > N=%lld)", bits, P->N);
    }
    nd[q] = n;
  }
  ht_mark("validate");
  const size_t head = 2 * ((size_t)nops + 1);  // long long offsets, in u32 words
  const size_t dmax = (size_t)((P->N + digit_bits - 1) / digit_bits);
  const size_t cap = head + (size_t)nops * dmax;
  const size_t prw = (size_t)batch * P->prod_limbs;
  int rc;
  if ((rc = ensure_pin(P, std::max(cap, prw)))) return rc;
  if (cap > P->stage_words) {
    P->dgraphs.clear();
    cudaFree(P->d_stage);
    P->d_stage = nullptr;
    CUCHK(cudaMalloc(&P->d_stage, cap * 4));
    P->stage_words = cap;
  }
  if (batch == 1 && !sq && nops == 2 && split_ok(P)) {
    if ((rc = run_digits_split(P, nd, ptrs, digit_bits, head))) return rc;
  } else {
    auto key = std::make_tuple(batch, sq, digit_bits);
    auto* ent = P->dgraphs.find(key);
    if (!ent) {
      if ((rc = tc_prepare(P, batch, sq))) return rc;
      cudaStream_t cap_s;
      CUCHK(cudaStreamCreateWithFlags(&cap_s, cudaStreamNonBlocking));
      CUCHK(cudaStreamBeginCapture(cap_s, cudaStreamCaptureModeThreadLocal));
      {
        CaptureScope cs;
        RepackArgs R{};
        R.stage = P->d_stage + head;
        R.off = reinterpret_cast<const long long*>(P->d_stage);
        R.dst = P->d_ops;
        R.ndst = P->op_limbs;
        R.sbits = digit_bits;
        const int gx = (int)std::max<long long>(1, std::min<long long>((P->op_limbs + 255) / 256, 1184 / nops + 1));
        launch_k(k_repack_bits, dim3(gx, nops), dim3(256), 0, cap_s, R);
        const uint32_t* bo = sq ? nullptr : P->d_ops + (size_t)batch * P->op_limbs;
        rc = run_mul(P, batch, P->d_ops, bo, P->op_limbs, P->d_prod, cap_s);
      }
      cudaGraph_t g;
      cudaError_t e = cudaStreamEndCapture(cap_s, &g);
      cudaStreamDestroy(cap_s);
      if (rc) {
        if (e == cudaSuccess) cudaGraphDestroy(g);
        return rc;
      }
      if (e != cudaSuccess) return fail(DKSS_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
      if (!(ent = P->dgraphs.put(key, g, &e))) return fail(DKSS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
    }
    long long* off = reinterpret_cast<long long*>(P->h_pin);
    uint32_t* dig = P->h_pin + head;
    long long o = 0;
    for (int q = 0; q < nops; ++q) {
      off[q] = o;
      o += (long long)nd[q];
    }
    off[nops] = o;
    if (nops <= 4) {
      // few operands: the header from the staging buffer, the digits straight from the caller's
      // pageable memory (the driver pipelines its own staging with the DMA, run_digits_split)
      CUCHK(cudaMemcpyAsync(P->d_stage, P->h_pin, head * 4, cudaMemcpyHostToDevice, P->stream));
      for (int q = 0; q < nops; ++q)
        if (nd[q])
          CUCHK(cudaMemcpyAsync(P->d_stage + head + off[q], ptrs[q], nd[q] * 4, cudaMemcpyHostToDevice, P->stream));
    } else {
      host_par((size_t)nops, (size_t)o * 4, [&](size_t q) {
        if (nd[q]) memcpy(dig + off[q], ptrs[q], nd[q] * 4);
      });
      CUCHK(cudaMemcpyAsync(P->d_stage, P->h_pin, (head + (size_t)o) * 4, cudaMemcpyHostToDevice, P->stream));
    }
    ht_mark("stage_copy");
    CUCHK(P->dgraphs.launch(ent, P->stream));
    ht_mark("graph_launch");
  }
  if (g_ht && g_ht->on) {  // timing study (experiment builds): the graph alone
    CUCHK(cudaStreamSynchronize(P->stream));
    ht_mark("graph_sync");
  }
  const size_t ncopy = std::min<size_t>(nc, P->prod_limbs);
  std::vector<char> over((size_t)batch, 0);
  if (nc >= (size_t)P->prod_limbs && is_pinned(c)) {
    // pinned destination (dkss_host_alloc): the products come straight from the device
    if (nc == (size_t)P->prod_limbs)
      CUCHK(cudaMemcpyAsync(c, P->d_prod, prw * 4, cudaMemcpyDeviceToHost, P->stream));
    else
      CUCHK(cudaMemcpy2DAsync(c, nc * 4, P->d_prod, P->prod_limbs * 4, P->prod_limbs * 4, batch,
                              cudaMemcpyDeviceToHost, P->stream));
    CUCHK(cudaStreamSynchronize(P->stream));
    ht_mark("sync_d2h_direct");
    if (nc > ncopy)
      for (int i = 0; i < batch; ++i) memset(c + (size_t)i * nc + ncopy, 0, (nc - ncopy) * 4);
  } else {
    CUCHK(cudaMemcpyAsync(P->h_pin, P->d_prod, prw * 4, cudaMemcpyDeviceToHost, P->stream));
    CUCHK(cudaStreamSynchronize(P->stream));
    ht_mark("sync");
    auto row = [&](size_t i) {
      const uint32_t* src = P->h_pin + i * P->prod_limbs;
      uint32_t* dst = c + i * nc;
      if (batch == 1)
        par_memcpy(dst, src, ncopy * 4);
      else
        memcpy(dst, src, ncopy * 4);
      for (size_t k = ncopy; k < (size_t)P->prod_limbs; ++k)
        if (src[k]) over[i] = 1;
      if (nc > ncopy) memset(dst + ncopy, 0, (nc - ncopy) * 4);
    };
    if (batch == 1)
      row(0);
    else
      host_par((size_t)batch, prw * 4, row);
    ht_mark("copy_out");
  }
  for (int i = 0; i < batch; ++i)
    if (over[i]) return fail(DKSS_ERANGE, "product %d does not fit nc=%zu limbs", i, nc);
  return DKSS_OK;
}
}  // namespace

extern "C" {

int dkss_mul_batch_digits(dkss_plan* P, int batch, const uint32_t* const* a, const size_t* na,
                          const uint32_t* const* b, const size_t* nb, int digit_bits, uint32_t* c, size_t nc) {
  if (!P || batch < 1 || !a || !na || !b || !nb || !c) return fail(DKSS_EINVAL, "bad argument");
  const bool trusted = digit_bits & DKSS_DIGITS_TRUSTED;
  digit_bits &= ~DKSS_DIGITS_TRUSTED;
  if (digit_bits < 8 || digit_bits > 32) return fail(DKSS_EINVAL, "digit_bits=%d outside [8, 32]", digit_bits);
  if (2LL * batch > 65535) return fail(DKSS_EINVAL, "batch %d too large", batch);
  bool sq = true;  // every pair is (x, x): square (one forward transform)
  for (int i = 0; i < batch && sq; ++i) sq = a[i] == b[i] && na[i] == nb[i];
  const int nops = (sq ? 1 : 2) * batch;
  std::vector<const uint32_t*> ptrs((size_t)nops);
  std::vector<size_t> counts((size_t)nops);
  for (int i = 0; i < batch; ++i) {
    ptrs[i] = a[i];
    counts[i] = na[i];
    if (!sq) {
      ptrs[batch + i] = b[i];
      counts[batch + i] = nb[i];
    }
  }
  size_t total = 2 * ((size_t)nops + 1);
  for (size_t q = 0; q < counts.size(); ++q) total += counts[q];
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, batch))) return rc;
  // staging sized once for both directions: it must not be reallocated while a copy is in flight
  if ((rc = ensure_pin(P, std::max<size_t>(total, (size_t)batch * (size_t)P->prod_limbs)))) return rc;
  HostTimer ht;
  g_ht = &ht;
  rc = run_digits_graph(P, batch, sq, nops, ptrs.data(), counts.data(), digit_bits, trusted, c, nc);
  g_ht = nullptr;
  return rc;
}

int dkss_host_alloc(size_t bytes, void** out) {
  if (!out || !bytes) return fail(DKSS_EINVAL, "bad argument");
  *out = nullptr;
  auto& pool = pinned_pool();
  {
    std::lock_guard<std::mutex> lk(pool.mu);
    auto it = pool.free_.lower_bound(bytes);
    if (it != pool.free_.end() && it->first <= 2 * bytes) {  // reuse a block of up to twice the size
      *out = it->second;
      pool.cached -= it->first;
      pool.live[it->second] = it->first;
      pool.free_.erase(it);
      return DKSS_OK;
    }
  }
  void* p = nullptr;
  CUCHK(cudaMallocHost(&p, bytes));
  std::lock_guard<std::mutex> lk(pool.mu);
  pool.live[p] = bytes;
  *out = p;
  return DKSS_OK;
}

void dkss_host_free(void* p) {
  if (!p) return;
  auto& pool = pinned_pool();
  std::lock_guard<std::mutex> lk(pool.mu);
  auto it = pool.live.find(p);
  if (it == pool.live.end()) return;  // not ours
  const size_t bytes = it->second;
  pool.live.erase(it);
  pool.free_.emplace(bytes, p);
  pool.cached += bytes;
  while (pool.cached > PinnedPool::kCacheCap && !pool.free_.empty()) {  // release the largest blocks
    auto big = std::prev(pool.free_.end());
    pool.cached -= big->first;
    cudaFreeHost(big->second);
    pool.free_.erase(big);
  }
}

int dkss_mul_digits(dkss_plan* P, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, int digit_bits,
                    uint32_t* c, size_t nc) {
  return dkss_mul_batch_digits(P, 1, &a, &na, &b, &nb, digit_bits, c, nc);
}

int dkss_mul(dkss_plan* P, const uint32_t* a, size_t na, const uint32_t* b, size_t nb, uint32_t* c, size_t nc) {
  if (!P || !a || !b || !c) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)na > P->op_limbs || (long long)nb > P->op_limbs) {
    // allow zero high limbs beyond the plan
    size_t na2 = na, nb2 = nb;
    while (na2 > 0 && (long long)na2 > P->op_limbs && a[na2 - 1] == 0) --na2;
    while (nb2 > 0 && (long long)nb2 > P->op_limbs && b[nb2 - 1] == 0) --nb2;
    if ((long long)na2 > P->op_limbs || (long long)nb2 > P->op_limbs)
      return fail(DKSS_ERANGE, "operand does not fit the plan");
    na = na2;
    nb = nb2;
  }
  std::vector<uint32_t> A((size_t)P->op_limbs, 0), B((size_t)P->op_limbs, 0);
  memcpy(A.data(), a, na * 4);
  memcpy(B.data(), b, nb * 4);
  return dkss_mul_batch(P, 1, A.data(), B.data(), (size_t)P->op_limbs, c, nc);
}

// --- four-step split of one multiply over `world` ranks -------------
// The first transform level is the reference's column step (bigmul/dkss.py:471-492): with
// E = 2m and mu0 = 2M/E, rank r owns global columns [r*C, (r+1)*C), C = mu0/world, held as
// [E][C] elements. Every deeper level and the bottom stay inside one of the E rows of mu0
// elements (bigmul/dkss.py:493-495), so after one exchange rank h owns rows [h*R, (h+1)*R),
// R = E/world, as [R][mu0]. The inverse walks the same split backwards.
namespace {
int fs_check(const dkss_plan* P, int rank, int world) {
  if (!P) return fail(DKSS_EINVAL, "bad argument");
  const long long E = 2LL * P->m, mu0 = 1LL << P->log_top_mu;
  if (world < 1 || (world & (world - 1)) || world > E || mu0 % world)
    return fail(DKSS_EINVAL, "world=%d must be a power of 2 dividing 2m=%lld and mu0=%lld", world, E, mu0);
  if (rank < 0 || rank >= world) return fail(DKSS_EINVAL, "rank %d outside [0, %d)", rank, world);
  if (P->levels < 1) return fail(DKSS_EINVAL, "plan has a single transform level; nothing to split");
  return 0;
}
}  // namespace

int dkss_fs_layout_get(const dkss_plan* P, int world, dkss_fs_layout* o) {
  int rc;
  if ((rc = fs_check(P, 0, world))) return rc;
  if (!o) return fail(DKSS_EINVAL, "bad argument");
  const long long mu0 = 1LL << P->log_top_mu;
  o->cols = mu0 / world;
  o->rows = 2LL * P->m / world;
  o->elem_words = (long long)P->m * P->L;
  o->block_words = P->poly_words / world;
  o->decode_seg = P->u == 32 ? o->cols * (P->m / 2) + P->m / 2 + P->L - 1 : 0;
  return DKSS_OK;
}

int dkss_fs_decode_partial(dkss_plan* P, int rank, int world, const uint32_t* x, uint64_t* s_out, void* stream) {
  int rc;
  if ((rc = fs_check(P, rank, world))) return rc;
  if (!x || !s_out) return fail(DKSS_EINVAL, "bad argument");
  if (P->u != 32) return fail(DKSS_EINVAL, "distributed decode needs u = 32 (plan has u = %d)", P->u);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  PartialArgs A{};
  A.x = x;
  A.s_out = reinterpret_cast<unsigned long long*>(s_out);
  A.C = (1LL << P->log_top_mu) / world;
  A.seg = A.C * (P->m / 2) + P->m / 2 + P->L - 1;
  A.mu0 = 1LL << P->log_top_mu;
  A.twoM = 2LL * P->M;
  A.rank = rank;
  A.E = 2 * P->m;
  A.MM = P->m;
  A.L = P->L;
  const long long total = (long long)(A.E + 1) * A.seg;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  launch_k(k_decode_partial, dim3(grid), dim3(256), 0, (cudaStream_t)stream, A);
  CUCHK(cudaGetLastError());
  return DKSS_OK;
}

int dkss_fs_decode_finish(dkss_plan* P, int world, const uint64_t* parts, uint32_t* out, size_t nc, void* stream) {
  int rc;
  if ((rc = fs_check(P, 0, world))) return rc;
  if (!parts || !out) return fail(DKSS_EINVAL, "bad argument");
  if (P->u != 32) return fail(DKSS_EINVAL, "distributed decode needs u = 32 (plan has u = %d)", P->u);
  if ((long long)nc < P->prod_limbs) return fail(DKSS_EINVAL, "nc=%zu below product limbs %lld", nc, P->prod_limbs);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  if ((rc = ensure_ws(P, 1))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (!P->d_sglob) CUCHK(cudaMalloc(&P->d_sglob, (size_t)P->prod_limbs * 8));
  CUCHK(cudaMemsetAsync(P->d_sglob, 0, (size_t)P->prod_limbs * 8, s));
  AssembleArgs A{};
  A.parts = reinterpret_cast<const unsigned long long*>(parts);
  A.sglob = P->d_sglob;
  A.C = (1LL << P->log_top_mu) / world;
  A.seg = A.C * (P->m / 2) + P->m / 2 + P->L - 1;
  A.nout = P->prod_limbs;
  A.mu0 = 1LL << P->log_top_mu;
  A.twoM = 2LL * P->M;
  A.world = world;
  A.E = 2 * P->m;
  A.half = P->m / 2;
  const long long total = (long long)world * (A.E + 1) * A.seg;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  launch_k(k_decode_assemble, dim3(grid), dim3(256), 0, s, A);
  CUCHK(cudaGetLastError());
  if ((rc = launch_decode(P, nullptr, out, 1, s, P->d_sglob))) return rc;
  if ((long long)nc > P->prod_limbs)
    CUCHK(cudaMemsetAsync(out + P->prod_limbs, 0, ((long long)nc - P->prod_limbs) * 4, s));
  return DKSS_OK;
}

namespace {
int fs_columns_fwd(dkss_plan* P, int rank, int world, const uint32_t* a, const uint32_t* b, size_t nl, uint32_t* x,
                   const uint64_t* z_peers, void* stream) {
  int rc;
  if ((rc = fs_check(P, rank, world))) return rc;
  if (!a || !b || !x) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nl > P->op_limbs) return fail(DKSS_ERANGE, "operand limbs %zu exceed plan (%lld)", nl, P->op_limbs);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  const int logC = P->log_top_mu - ilog2i(world);
  Geom g{P->poly_words / world, logC, (long long)rank << logC, logC};
  if (z_peers) {  // outputs straight into the row owners' [2][R][mu0] buffers
    g.peer = reinterpret_cast<const unsigned long long*>(z_peers);
    g.peer_mode = 1;
    g.peer_log_r = ilog2i(2LL * P->m / world);
    g.peer_log_c = logC;
    g.peer_log_mu0 = P->log_top_mu;
  }
  return launch_fwd_levels(P, x, 2, (cudaStream_t)stream, a, b, (long long)nl, 1, 0, 1, &g);
}

int fs_rows(dkss_plan* P, int rank, int world, uint32_t* z, const uint64_t* x_peers, void* stream) {
  int rc;
  if ((rc = fs_check(P, rank, world))) return rc;
  if (!z) return fail(DKSS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int rows = 2 * P->m / world;
  const long long row_words = P->poly_words / (2LL * P->m);
  const long long f_items = 2LL * rows << (P->log_top_mu - P->logE);
  if (!x_peers && P->dyn_grid && f_items >= 2LL * P->dyn_grid) {
    // the persistent row-phase kernel on this rank's R rows of a and b when there are enough
    // column items to keep its grid busy (2^26 on 8 ranks: 0.43 vs 0.50 ms; 2^24 on 8 ranks,
    // 256 items: the three launches win); its counters live in the plan workspace
    if ((rc = ensure_ws(P, 1))) return rc;
    return launch_dyn(P, z, z + (size_t)rows * row_words, 1, false, s, rows);
  }
  Geom g{row_words, P->log_top_mu - P->logE, 0, -1};
  if ((rc = launch_fwd_levels(P, z, 2 * rows, s, nullptr, nullptr, 0, 0, 1, P->levels, &g))) return rc;
  BottomArgs A{};
  A.a = z;
  A.b = z + (size_t)rows * row_words;
  A.poly_words = row_words;
  A.elems_per_poly = 1LL << P->log_top_mu;
  A.logb = P->logb;
  A.mode = 1;
  A.scale = 0;
  A.total_elems = (long long)rows << P->log_top_mu;
  const int grid = (int)std::min<long long>((A.total_elems + P->kt.ne - 1) / P->kt.ne, P->grid_bot);
  A.ctr = next_tick(P, (A.total_elems + P->kt.ne - 1) / P->kt.ne, grid);
  launch_k(P->kt.bottom, dim3(grid), dim3(P->kt.nt), smem_two(P), s, A, P->mc);
  CUCHK(cudaGetLastError());
  mark(P, s, DKSS_K_BOTTOM, rp_work(P, A.total_elems), 3LL * A.total_elems * P->m * P->L * 4);
  if (x_peers) {  // the last inverse level stores the product rows into the column owners' [E][C]
    g.peer = reinterpret_cast<const unsigned long long*>(x_peers);
    g.peer_mode = 2;
    g.peer_log_c = P->log_top_mu - ilog2i(world);
    g.peer_row0 = (long long)rank * rows;
  }
  return launch_inv_levels(P, z, rows, false, s, 1, P->levels, &g);
}
}  // namespace

int dkss_fs_columns_fwd(dkss_plan* P, int rank, int world, const uint32_t* a, const uint32_t* b, size_t nl,
                        uint32_t* x, void* stream) {
  return fs_columns_fwd(P, rank, world, a, b, nl, x, nullptr, stream);
}

int dkss_fs_columns_fwd_peer(dkss_plan* P, int rank, int world, const uint32_t* a, const uint32_t* b, size_t nl,
                             uint32_t* x, const uint64_t* z_peers, void* stream) {
  if (!z_peers) return fail(DKSS_EINVAL, "bad argument");
  return fs_columns_fwd(P, rank, world, a, b, nl, x, z_peers, stream);
}

int dkss_fs_rows(dkss_plan* P, int world, uint32_t* z, void* stream) { return fs_rows(P, 0, world, z, nullptr, stream); }

int dkss_fs_rows_peer(dkss_plan* P, int rank, int world, uint32_t* z, const uint64_t* x_peers, void* stream) {
  if (!x_peers) return fail(DKSS_EINVAL, "bad argument");
  if (P && P->levels < 2) return fail(DKSS_EINVAL, "fused exchange needs two or more transform levels");
  return fs_rows(P, rank, world, z, x_peers, stream);
}

int dkss_ipc_alloc(int device, size_t bytes, void** dptr, void* handle) {
  if (!dptr || !handle || !bytes) return fail(DKSS_EINVAL, "bad argument");
  CUCHK(cudaSetDevice(device));
  CUCHK(cudaMalloc(dptr, bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
  if (e != cudaSuccess) {
    cudaFree(*dptr);
    *dptr = nullptr;
    return fail(DKSS_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  memcpy(handle, &h, sizeof h);
  return DKSS_OK;
}

int dkss_ipc_open(int device, const void* handle, void** dptr) {
  if (!dptr || !handle) return fail(DKSS_EINVAL, "bad argument");
  CUCHK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  CUCHK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DKSS_OK;
}

int dkss_ipc_close(void* dptr) {
  if (!dptr) return DKSS_OK;
  CUCHK(cudaIpcCloseMemHandle(dptr));
  return DKSS_OK;
}

int dkss_ipc_free(void* dptr) {
  if (!dptr) return DKSS_OK;
  CUCHK(cudaFree(dptr));
  return DKSS_OK;
}

int dkss_fs_columns_inv(dkss_plan* P, int rank, int world, uint32_t* x, void* stream) {
  int rc;
  if ((rc = fs_check(P, rank, world))) return rc;
  if (!x) return fail(DKSS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  const int logC = P->log_top_mu - ilog2i(world);
  const Geom g{P->poly_words / world, logC, (long long)rank << logC, logC};
  return launch_inv_levels(P, x, 1, true, (cudaStream_t)stream, 0, 1, &g);
}

int dkss_block_transpose(dkss_plan* P, const uint32_t* src, uint32_t* dst, int n, int A, int B, int64_t run_words,
                         void* stream) {
  if (!P || !src || !dst || n < 1 || A < 1 || B < 1 || run_words < 4 || (run_words & 3) || src == dst)
    return fail(DKSS_EINVAL, "bad argument");
  if (((uintptr_t)src | (uintptr_t)dst) & 15) return fail(DKSS_EINVAL, "buffers must be 16-byte aligned");
  if ((long long)n * A * B > 65535) return fail(DKSS_EINVAL, "too many blocks");
  CUCHK(cudaSetDevice(P->device));
  const long long run = run_words / 4;
  const int gx = (int)std::max<long long>(1, std::min<long long>((run + 255) / 256, std::max(1, 1184 / (n * A * B))));
  count_launch();
  k_block_transpose<<<dim3(gx, n * A * B), 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, A, B, run);
  CUCHK(cudaGetLastError());
  mark(P, (cudaStream_t)stream, DKSS_K_TRANSPOSE, 0, 2LL * n * A * B * run_words * 4);
  return DKSS_OK;
}

int dkss_decode_device(dkss_plan* P, const uint32_t* v, uint32_t* out, size_t nc, void* stream) {
  if (!P || !v || !out) return fail(DKSS_EINVAL, "bad argument");
  if ((long long)nc < P->prod_limbs) return fail(DKSS_EINVAL, "nc=%zu below product limbs %lld", nc, P->prod_limbs);
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, 1))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if ((rc = launch_decode(P, v, out, 1, s))) return rc;
  if ((long long)nc > P->prod_limbs)
    CUCHK(cudaMemsetAsync(out + P->prod_limbs, 0, ((long long)nc - P->prod_limbs) * 4, s));
  return DKSS_OK;
}

// --- Lucas-Lehmer driver (bigmul/bench.py:197-217) -----------------------------------
namespace {
int ll_graph(dkss_plan* P, long long p, int k, GraphLru<std::pair<long long, int>>::Ent** out) {
  if ((*out = P->ll_graphs.find({p, k}))) return 0;
  int rc0;
  if ((rc0 = tc_prepare(P, 1, true))) return rc0;
  cudaStream_t cap;
  CUCHK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  CUCHK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  int rc = 0;
  {
    CaptureScope cs;
    MersArgs M{P->d_prod, P->prod_limbs, p, P->d_ops};
    for (int i = 0; i < k && !rc; ++i) {
      rc = run_mul(P, 1, P->d_ops, nullptr, P->op_limbs, P->d_prod, cap);
      if (!rc) launch_k(k_mersenne_sub2, dim3(1), dim3(kMersThreads), 0, cap, M);
    }
  }
  cudaGraph_t g;
  cudaError_t e = cudaStreamEndCapture(cap, &g);
  cudaStreamDestroy(cap);
  if (rc) {
    if (e == cudaSuccess) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(DKSS_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
  if (!(*out = P->ll_graphs.put({p, k}, g, &e)))
    return fail(DKSS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
  return 0;
}
}  // namespace

int dkss_lucas_lehmer(dkss_plan* P, int64_t p, int64_t iters, uint32_t* s, size_t ns) {
  if (!P || !s || iters < 0) return fail(DKSS_EINVAL, "bad argument");
  if (p < 2 || p > P->N) return fail(DKSS_EINVAL, "exponent p=%lld outside [2, N=%lld]", (long long)p, P->N);
  const size_t n = (size_t)((p + 31) / 32);
  if (ns < n) return fail(DKSS_EINVAL, "state needs %zu limbs, got %zu", n, ns);
  for (size_t i = n; i < ns; ++i)
    if (s[i]) return fail(DKSS_ERANGE, "state exceeds 2^p");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, 1))) return rc;
  cudaStream_t st = P->stream;
  CUCHK(cudaMemsetAsync(P->d_ops, 0, P->op_limbs * 4, st));
  CUCHK(cudaMemcpyAsync(P->d_ops, s, n * 4, cudaMemcpyHostToDevice, st));
  const int K = 16;
  long long left = iters;
  while (left > 0) {
    const int k = left >= K ? K : (int)left;
    GraphLru<std::pair<long long, int>>::Ent* ge;
    if ((rc = ll_graph(P, p, k, &ge))) return rc;
    CUCHK(P->ll_graphs.launch(ge, st));
    left -= k;
  }
  CUCHK(cudaMemcpyAsync(s, P->d_ops, n * 4, cudaMemcpyDeviceToHost, st));
  CUCHK(cudaStreamSynchronize(st));
  return DKSS_OK;
}

int dkss_encode_host(dkss_plan* P, const uint32_t* a, size_t na, uint32_t* poly) {
  if (!P || !a || !poly) return fail(DKSS_EINVAL, "bad argument");
  int rc;
  if ((rc = check_operand(P, a, na))) return rc;
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  if ((rc = ensure_ws(P, 1))) return rc;
  size_t nl = std::min<size_t>(na, (size_t)P->op_limbs);
  std::vector<uint32_t> A((size_t)P->op_limbs, 0);
  memcpy(A.data(), a, nl * 4);
  CUCHK(cudaMemcpyAsync(P->d_ops, A.data(), A.size() * 4, cudaMemcpyHostToDevice, P->stream));
  if ((rc = launch_encode(P, P->d_ops, P->op_limbs, P->d_poly, 1, P->stream))) return rc;
  CUCHK(cudaMemcpyAsync(poly, P->d_poly, P->poly_words * 4, cudaMemcpyDeviceToHost, P->stream));
  CUCHK(cudaStreamSynchronize(P->stream));
  return DKSS_OK;
}

int dkss_fft_host(dkss_plan* P, uint32_t* polys, int count) {
  if (!P || !polys || count < 1) return fail(DKSS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, count))) return rc;  // 2*count polys available
  uint32_t* work = P->d_poly;
  uint32_t* scratch = P->d_poly + (size_t)count * P->poly_words;
  const size_t bytes = (size_t)count * P->poly_words * 4;
  cudaStream_t s = P->stream;
  CUCHK(cudaMemcpyAsync(work, polys, bytes, cudaMemcpyHostToDevice, s));
  if ((rc = launch_fwd_levels(P, work, count, s))) return rc;
  if ((rc = launch_bottom(P, work, nullptr, count, 0, false, s))) return rc;
  const long long elems = 2LL * P->M;
  count_launch();
  k_permute<<<(int)std::min<long long>((elems * count * P->m * P->L + 255) / 256, 148LL * 32), 256, 0, s>>>(
      work, scratch, elems, P->m * P->L, P->logE, P->levels, P->logb, 1, P->poly_words, count);
  CUCHK(cudaGetLastError());
  CUCHK(cudaMemcpyAsync(polys, scratch, bytes, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  return DKSS_OK;
}

int dkss_rmul_host(dkss_plan* P, const uint32_t* x, const uint32_t* y, uint32_t* out, size_t count) {
  if (!P || !x || !y || !out) return fail(DKSS_EINVAL, "bad argument");
  if (count == 0) return DKSS_OK;
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  const size_t ew = (size_t)P->m * P->L;
  uint32_t *dx, *dy, *dout;
  CUCHK(cudaMalloc(&dx, count * ew * 4));
  CUCHK(cudaMalloc(&dy, count * ew * 4));
  CUCHK(cudaMalloc(&dout, count * ew * 4));
  cudaStream_t s = P->stream;
  cudaMemcpyAsync(dx, x, count * ew * 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dy, y, count * ew * 4, cudaMemcpyHostToDevice, s);
  const int grid = (int)((count + P->kt.ne - 1) / P->kt.ne);
  count_launch();
  P->kt.rmul<<<grid, P->kt.nt, P->kt.smem_rmul, s>>>(dx, dy, dout, (long long)count, P->mc);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, count * ew * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(dx);
  cudaFree(dy);
  cudaFree(dout);
  if (e != cudaSuccess) return fail(DKSS_ECUDA, "rmul failed: %s", cudaGetErrorString(e));
  return DKSS_OK;
}

int dkss_decode_host(dkss_plan* P, const uint32_t* v, uint32_t* out, size_t nout) {
  if (!P || !v || !out) return fail(DKSS_EINVAL, "bad argument");
  std::lock_guard<std::mutex> lk(P->mu);
  CUCHK(cudaSetDevice(P->device));
  int rc;
  if ((rc = ensure_ws(P, 1))) return rc;
  cudaStream_t s = P->stream;
  CUCHK(cudaMemcpyAsync(P->d_poly, v, P->poly_words * 4, cudaMemcpyHostToDevice, s));
  const long long nres = 2LL * P->M * P->m;
  count_launch();
  P->kt.mscale<<<(int)std::min<long long>((nres + 255) / 256, 4096), 256, 0, s>>>(P->d_poly, nres, 1, P->mc);
  CUCHK(cudaGetLastError());
  if ((rc = launch_decode(P, P->d_poly, P->d_prod, 1, s))) return rc;
  std::vector<uint32_t> full((size_t)P->prod_limbs);
  CUCHK(cudaMemcpyAsync(full.data(), P->d_prod, full.size() * 4, cudaMemcpyDeviceToHost, s));
  CUCHK(cudaStreamSynchronize(s));
  const size_t ncopy = std::min<size_t>(nout, full.size());
  memcpy(out, full.data(), ncopy * 4);
  for (size_t k = ncopy; k < full.size(); ++k)
    if (full[k]) return fail(DKSS_ERANGE, "decoded value does not fit nout=%zu limbs", nout);
  if (nout > ncopy) memset(out + ncopy, 0, (nout - ncopy) * 4);
  return DKSS_OK;
}

}  // extern "C"

// Schoenhage-Strassen multiply (include/smul.h)
#include "smul_capi.cuh"
