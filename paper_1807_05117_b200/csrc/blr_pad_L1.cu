// blr_pad_L1.cu — explicit instantiation of the pad-engine launchers for
// line length 1 = 1 x 1 (one translation unit per length: parallel build).
#include "blr_pad_kernels.cuh"

namespace blr {
template void launch_xinv<double, WShape<1, 1>>(blr_ctx*, PadEngine*, const XPassArgs<double>&);
template void launch_yinv<double, WShape<1, 1>>(blr_ctx*, PadEngine*, const YPassArgs<double>&);
template void launch_yfwd<double, WShape<1, 1>>(blr_ctx*, PadEngine*, const YFwdArgs<double>&);
template void launch_xfwd<double, WShape<1, 1>>(blr_ctx*, PadEngine*, const FwdArgs<double>&);
template void launch_xinv<float, WShape<1, 1>>(blr_ctx*, PadEngine*, const XPassArgs<float>&);
template void launch_yinv<float, WShape<1, 1>>(blr_ctx*, PadEngine*, const YPassArgs<float>&);
template void launch_yfwd<float, WShape<1, 1>>(blr_ctx*, PadEngine*, const YFwdArgs<float>&);
template void launch_xfwd<float, WShape<1, 1>>(blr_ctx*, PadEngine*, const FwdArgs<float>&);
}  // namespace blr
