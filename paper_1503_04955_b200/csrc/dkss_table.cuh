// dkss_table.cuh -- per-(m, L) kernel table; each m is instantiated in its own
// translation unit (dkss_inst_m*.cu) so the build parallelises.
#pragma once
#include "dkss_kernels.cuh"
#include "dkss_warp.cuh"
#include "dkss_rows.cuh"
#include "dkss_dyn.cuh"
#include "dkss_tc.cuh"

namespace dkss {

struct KTable {
  void (*fwd)(PassArgs, ModCtx);
  void (*inv)(PassArgs, ModCtx);
  // DFT-only passes (table twiddles on the tensor cores), m in {16, 32}; else null
  void (*fwd_do)(PassArgs, ModCtx);
  void (*inv_do)(PassArgs, ModCtx);
  size_t smem_pass_do;
  int cols_do;  // columns per tile of the DFT-only passes (PCfg)
  void (*fwd_w)(PassArgs, ModCtx);  // warp-per-column variants (m <= 16), else null
  void (*inv_w)(PassArgs, ModCtx);
  size_t smem_fwd_w, smem_inv_w;    // dynamic shared memory per CTA (kWarpsPerCta warps)
  void (*dft)(PassArgs, ModCtx);    // split passes: column DFT (m <= 16) and elementwise twiddle
  void (*tw)(PassArgs, ModCtx);
  size_t smem_dft;
  void (*bottom)(BottomArgs, ModCtx);
  void (*rmul)(const uint32_t*, const uint32_t*, uint32_t*, long long, ModCtx);
  void (*mscale)(uint32_t*, long long, int, ModCtx);
  void (*build_twr)(const uint32_t*, uint32_t*, long long, int, ModCtx);
  int ne;     // elements per CTA
  int cols;   // columns per CTA
  int nt;             // threads per CTA
  size_t smem_pass;   // dynamic shared memory bytes: column passes
  size_t smem_bot;    // bottom kernel
  size_t smem_rmul;   // standalone ring product
  // row phase of two-level plans in one cluster kernel (dkss_rows.cuh), by cluster size
  // CS = base length b in {2, 4, 8, 16}; null where not instantiated
  void (*rows[5])(RowsArgs, ModCtx);
  size_t smem_rows;
  // row phase of two-level plans as one persistent kernel with dependency-driven items
  // (dkss_dyn.cuh); null for m = 8
  void (*dyn)(DynArgs, ModCtx);
  size_t smem_dyn;
  // twiddle products on the tensor cores (dkss_tc.cuh): m in {16, 32}, L = 4 only, else null
  void (*tc)(TcArgs);
  void (*tc_build)(const uint32_t*, long long, uint8_t*, ModCtx, const uint32_t*);
  size_t smem_tc;
  size_t tc_vbytes;  // bytes of one V table row set (per twiddle row s)
};

template <int MM, int L>
KTable make_table() {
  KTable t{};
  t.fwd = k_fwd_pass<MM, L>;
  t.inv = k_inv_pass<MM, L>;
  if constexpr (MM == 32 || MM == 16) {
    using PC = PCfg<MM, true>;
    static_assert(!PC::TWS, "DFT-only passes stage no twiddle rows");
    t.fwd_do = k_fwd_pass<MM, L, true>;
    t.inv_do = k_inv_pass<MM, L, true>;
    t.smem_pass_do = 2 * PC::NE * Smem<MM, L>::ES * 4;  // two stages; the register DFT needs no ping-pong
    t.cols_do = PC::COLS;
  }
  t.tw = k_twiddle<MM, L>;
  if constexpr (MM <= 16) {
    t.fwd_w = k_fwd_warp<MM, L>;
    t.inv_w = k_inv_warp<MM, L>;
    t.smem_fwd_w = (size_t)kWarpsPerCta * 2 * MM * Smem<MM, L>::ES * 4;
    t.smem_inv_w = 2 * t.smem_fwd_w;
    t.dft = k_dft_cols<MM, L>;
    t.smem_dft = t.smem_fwd_w;
  } else {
    t.fwd_w = t.inv_w = nullptr;
    t.smem_fwd_w = t.smem_inv_w = 0;
  }
  t.bottom = k_bottom<MM, L>;
  if constexpr (MM == 16 || MM == 32) {
    t.rows[1] = k_rows<MM, L, 2>;
    t.rows[2] = k_rows<MM, L, 4>;
    t.rows[3] = k_rows<MM, L, 8>;
    t.rows[4] = k_rows<MM, L, 16>;
    t.smem_rows = RowsSmem<MM, L>::WORDS * 4;
    if constexpr (Cfg<MM>::NE == 2 * MM) {  // one column per work item
      t.dyn = k_rows_dyn<MM, L>;
      t.smem_dyn = DynSmem<MM, L>::WORDS * 4;
    }
  }
  if constexpr (L == 4 && (MM == 16 || MM == 32)) {
    t.tc = k_tc_twiddle<MM>;
    t.tc_build = k_tc_build_v<MM>;
    t.smem_tc = TcSmem<MM>::BYTES;
    t.tc_vbytes = TcSmem<MM>::VBYTES;
  }
  t.rmul = k_rmul<MM, L>;
  t.mscale = k_mont_scale<L>;
  t.build_twr = k_build_twr<L>;
  t.ne = Cfg<MM>::NE;
  t.cols = Cfg<MM>::COLS;
  t.nt = Cfg<MM>::NT;
  t.smem_pass = SmemPlan<MM, L>::PASS * 4;
  t.smem_bot = SmemPlan<MM, L>::BOT * 4;
  t.smem_rmul = SmemPlan<MM, L>::RMUL * 4;
  return t;
}

#define DKSS_FOR_EACH_INST(X) \
  X(8, 2) X(8, 3) X(8, 4) X(8, 5) X(8, 6) X(16, 2) X(16, 3) X(16, 4) X(16, 5) X(16, 6) \
  X(32, 2) X(32, 3) X(32, 4) X(32, 5) X(32, 6)

#define DKSS_DECLARE(MM, L) KTable dkss_table_m##MM##_L##L();
DKSS_FOR_EACH_INST(DKSS_DECLARE)
#undef DKSS_DECLARE

}  // namespace dkss
