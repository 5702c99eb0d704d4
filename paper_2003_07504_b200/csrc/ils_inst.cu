// Kernel instantiations.  build.py compiles this file once per -D selector
// so the heavy FFT templates build in parallel:
//   -DILS_INST_ROW_RT=<float|double>    runtime-planned row kernels
//   -DILS_INST_COL_RT=<float|double>    runtime-planned column kernel
//   -DILS_INST_ROW_SPEC=<id>            fp32 row kernel for ILS_ROW_SPECS entry id
//   -DILS_INST_COL_SPEC=<id>            fp32 column kernel for ILS_COL_SPECS entry id
//   -DILS_INST_COL2                     fp32 two-stage column kernels (ILS_COL2_SPECS)
//   -DILS_INST_COL3                     fp32 three-stage column kernels (ILS_COL3_SPECS)
#define ILS_DEFINE_LAUNCHERS
#include "ils_kernels.cuh"
#include "ils_rowroll.cuh"
#ifdef ILS_INST_COL2
#include "ils_col2.cuh"
#endif
#ifdef ILS_INST_COL3
#include "ils_col3.cuh"
#endif

namespace ils {
#ifdef ILS_INST_ROW_RT
template cudaError_t launch_row_impl<ILS_INST_ROW_RT, true, FftRt>(const RowArgs<ILS_INST_ROW_RT>&, dim3, int, size_t,
                                                                   cudaStream_t);
template cudaError_t launch_row_impl<ILS_INST_ROW_RT, false, FftRt>(const RowArgs<ILS_INST_ROW_RT>&, dim3, int, size_t,
                                                                    cudaStream_t);
template cudaError_t launch_row_impl<ILS_INST_ROW_RT, true, FftRt, true>(const RowArgs<ILS_INST_ROW_RT>&, dim3, int,
                                                                         size_t, cudaStream_t);
#endif
#ifdef ILS_INST_COL_RT
template cudaError_t launch_col_impl<ILS_INST_COL_RT, FftRt>(const ColArgs<ILS_INST_COL_RT>&, dim3, int, size_t,
                                                             cudaStream_t);
template cudaError_t launch_col_impl<ILS_INST_COL_RT, FftRtWide>(const ColArgs<ILS_INST_COL_RT>&, dim3, int, size_t,
                                                                 cudaStream_t);
#endif
#ifdef ILS_INST_ROW_SPEC
template cudaError_t launch_row_impl<float, true, RowSpec<ILS_INST_ROW_SPEC>::type,
                                     ILS_ROW_SPEC_WIDE(ILS_INST_ROW_SPEC)>(const RowArgs<float>&, dim3, int, size_t,
                                                                            cudaStream_t);
#if ILS_ROW_SPEC_ROLL(ILS_INST_ROW_SPEC)
template cudaError_t launch_row_roll_impl<RowSpec<ILS_INST_ROW_SPEC>::type>(const RowArgs<float>&, dim3, size_t,
                                                                           int, cudaStream_t);
#endif
#endif
#ifdef ILS_INST_COL_SPEC
template cudaError_t launch_col_impl<float, ColSpec<ILS_INST_COL_SPEC>::type>(const ColArgs<float>&, dim3, int, size_t,
                                                                              cudaStream_t);
#endif
#ifdef ILS_INST_COL2
#define ILS_CASE(ID, N1, N2, CW, MINB) \
  template cudaError_t launch_col2_impl<N1, N2, CW, MINB>(const ColArgs<float>&, int, cudaStream_t);
ILS_COL2_SPECS(ILS_CASE)
#undef ILS_CASE
#endif
#ifdef ILS_INST_COL3
#define ILS_CASE(ID, N1, N2, N3, CW, MINB) \
  template cudaError_t launch_col3_impl<N1, N2, N3, CW, MINB>(const ColArgs<float>&, int, cudaStream_t);
ILS_COL3_SPECS(ILS_CASE)
#undef ILS_CASE
#endif
}  // namespace ils
