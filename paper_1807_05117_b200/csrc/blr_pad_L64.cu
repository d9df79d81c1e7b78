// blr_pad_L64.cu — explicit instantiation of the pad-engine launchers for
// line length 64 = 8 x 8 (one translation unit per length: parallel build).
#include "blr_pad_kernels.cuh"

namespace blr {
template void launch_xinv<double, WShape<8, 8>>(blr_ctx*, PadEngine*, const XPassArgs<double>&);
template void launch_yinv<double, WShape<8, 8>>(blr_ctx*, PadEngine*, const YPassArgs<double>&);
template void launch_yfwd<double, WShape<8, 8>>(blr_ctx*, PadEngine*, const YFwdArgs<double>&);
template void launch_xfwd<double, WShape<8, 8>>(blr_ctx*, PadEngine*, const FwdArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 0>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 1>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 2>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 3>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 4>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 5>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 6>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 7>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_lines<double, WShape<8, 8>, 8>(blr_ctx*, PadEngine*, const LineArgs<double>&);
template void launch_xinv<float, WShape<8, 8>>(blr_ctx*, PadEngine*, const XPassArgs<float>&);
template void launch_yinv<float, WShape<8, 8>>(blr_ctx*, PadEngine*, const YPassArgs<float>&);
template void launch_yfwd<float, WShape<8, 8>>(blr_ctx*, PadEngine*, const YFwdArgs<float>&);
template void launch_xfwd<float, WShape<8, 8>>(blr_ctx*, PadEngine*, const FwdArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 0>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 1>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 2>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 3>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 4>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 5>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 6>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 7>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_lines<float, WShape<8, 8>, 8>(blr_ctx*, PadEngine*, const LineArgs<float>&);
template void launch_fwd2<double, WShape<8, 8>>(blr_ctx*, PadEngine*, const Fwd2Args<double>&, int, int);
template bool fwd2_fits<double, WShape<8, 8>>(const PadGeom&);
template void launch_fwd2<float, WShape<8, 8>>(blr_ctx*, PadEngine*, const Fwd2Args<float>&, int, int);
template bool fwd2_fits<float, WShape<8, 8>>(const PadGeom&);
}  // namespace blr
