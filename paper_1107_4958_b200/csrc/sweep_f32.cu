// sweep_f32.cu - instantiations of the sweep kernels for float sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_f32(Mode m, int k) { return sweep_ptr_for<float>(m, k); }
const void* sweep_ptr_stream_f32(int k) { return stream_ptr_for<float>(k); }
const void* sweep_ptr_stream_mc_f32(int k) { return stream_mc_ptr_for<float>(k); }
const void* sweep_ptr_stream_out_f32(int k) { return stream_out_ptr_for<float>(k); }
const void* sweep_ptr_fused_f32(int k, int ls) {
  if (ls == LS_SMALL) return fused_f32_ptr_for<LS_SMALL>(k);
  if (ls == LS_MID) return fused_f32_ptr_for<LS_MID>(k);
  return fused_f32_ptr_for<LS>(k);
}
}  // namespace sb
