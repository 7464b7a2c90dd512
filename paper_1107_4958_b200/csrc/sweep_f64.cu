// sweep_f64.cu - instantiations of the sweep kernels for double sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_f64(Mode m, int k) { return sweep_ptr_for<double>(m, k); }
}  // namespace sb
