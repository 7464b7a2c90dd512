// sweep_u8.cu - instantiations of the sweep kernels for uint8_t sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_u8(Mode m, int k) { return sweep_ptr_for<uint8_t>(m, k); }

// the int32-plane column sweep does not read the source: one instantiation
const void* sweep_ptr_cols(int k) {
  switch (k) {
    case 1: return (const void*)sweep_kernel<uint8_t, 1, Mode::ColsFromMid>;
    case 2: return (const void*)sweep_kernel<uint8_t, 2, Mode::ColsFromMid>;
    case 3: return (const void*)sweep_kernel<uint8_t, 3, Mode::ColsFromMid>;
    case 4: return (const void*)sweep_kernel<uint8_t, 4, Mode::ColsFromMid>;
    case 5: return (const void*)sweep_kernel<uint8_t, 5, Mode::ColsFromMid>;
    case 6: return (const void*)sweep_kernel<uint8_t, 6, Mode::ColsFromMid>;
    case 7: return (const void*)sweep_kernel<uint8_t, 7, Mode::ColsFromMid>;
    default: return (const void*)sweep_kernel<uint8_t, 8, Mode::ColsFromMid>;
  }
}
}  // namespace sb
