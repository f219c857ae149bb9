// One (m, L) instantiation of the DKSS kernels; compiled once per pair with
// -DINST_MM=<m> -DINST_L=<L> (see paper_1503_04955_b200/build.py) so the build runs in parallel.
#include "dkss_table.cuh"

#if !defined(INST_MM) || !defined(INST_L)
#error "compile with -DINST_MM=<m> -DINST_L=<L>"
#endif

#define DKSS_CAT2(MM, L) dkss_table_m##MM##_L##L
#define DKSS_CAT(MM, L) DKSS_CAT2(MM, L)

namespace dkss {
KTable DKSS_CAT(INST_MM, INST_L)() { return make_table<INST_MM, INST_L>(); }
}  // namespace dkss

#if defined(DKSS_TC_TRACE) && INST_MM == 32 && INST_L == 4
// experiment builds only: copy out the role time stamps of the last eight tensor-core launches
extern "C" int dkss_exp_tc_trace(unsigned long long* out, unsigned int* launches) {
  if (cudaMemcpyFromSymbol(out, dkss::g_tc_trace, sizeof(dkss::g_tc_trace)) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(launches, dkss::g_tc_launch, sizeof(unsigned int)) != cudaSuccess) return -1;
  return 0;
}
#endif
