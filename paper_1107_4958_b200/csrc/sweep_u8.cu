// sweep_u8.cu - instantiations of the sweep kernels for uint8_t sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_u8(Mode m, int k) { return sweep_ptr_for<uint8_t>(m, k); }

// the int32-plane column sweep does not read the source: one instantiation
const void* sweep_ptr_cols(int k) { return cols_ptr_for<>(k); }
const void* sweep_ptr_cols2(int k) { return cols2_ptr_for<>(k); }
const void* sweep_ptr_cols2s(int k) { return cols2s_ptr_for<>(k); }
const void* sweep_ptr_fused3(int k) { return fused3_ptr_for<>(k); }
const void* sweep_ptr_fused5(int k) { return fused5_ptr_for<>(k); }
const void* sweep_ptr_fusedp(int k) { return fusedp_ptr_for<>(k); }
}  // namespace sb
