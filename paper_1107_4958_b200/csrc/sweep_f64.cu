// sweep_f64.cu - instantiations of the sweep kernels for double sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_f64(Mode m, int k) { return sweep_ptr_for<double>(m, k); }
const void* sweep_ptr_stream_f64(int k) { return stream_ptr_for<double>(k); }
const void* sweep_ptr_stream_mc_f64(int k) { return stream_mc_ptr_for<double>(k); }
const void* sweep_ptr_stream_out_f64(int k) { return stream_out_ptr_for<double>(k); }
}  // namespace sb
