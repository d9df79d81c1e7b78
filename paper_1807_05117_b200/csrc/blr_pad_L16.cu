// blr_pad_L16.cu — explicit instantiation of the pad-engine launchers for
// line length 16 = 4 x 4 (one translation unit per length: parallel build).
#include "blr_pad_kernels.cuh"

namespace blr {
template void launch_xinv<double, WShape<4, 4>>(blr_ctx*, PadEngine*, const XPassArgs<double>&);
template void launch_yinv<double, WShape<4, 4>>(blr_ctx*, PadEngine*, const YPassArgs<double>&);
template void launch_yfwd<double, WShape<4, 4>>(blr_ctx*, PadEngine*, const YFwdArgs<double>&);
template void launch_xfwd<double, WShape<4, 4>>(blr_ctx*, PadEngine*, const FwdArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 0>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 1>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 2>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 3>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 4>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 5>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 6>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 7>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<4, 4>, 8>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_xinv<float, WShape<4, 4>>(blr_ctx*, PadEngine*, const XPassArgs<float>&);
template void launch_yinv<float, WShape<4, 4>>(blr_ctx*, PadEngine*, const YPassArgs<float>&);
template void launch_yfwd<float, WShape<4, 4>>(blr_ctx*, PadEngine*, const YFwdArgs<float>&);
template void launch_xfwd<float, WShape<4, 4>>(blr_ctx*, PadEngine*, const FwdArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 0>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 1>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 2>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 3>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 4>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 5>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 6>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 7>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<4, 4>, 8>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_fwd2<double, WShape<4, 4>>(blr_ctx*, PadEngine*, const Fwd2Args<double>&, int, int);
template bool fwd2_fits<double, WShape<4, 4>>(const PadGeom&);
template void launch_fwd2<float, WShape<4, 4>>(blr_ctx*, PadEngine*, const Fwd2Args<float>&, int, int);
template bool fwd2_fits<float, WShape<4, 4>>(const PadGeom&);
}  // namespace blr
