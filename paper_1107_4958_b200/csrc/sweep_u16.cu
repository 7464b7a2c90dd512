// sweep_u16.cu - instantiations of the sweep kernels for uint16_t sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_u16(Mode m, int k) { return sweep_ptr_for<uint16_t>(m, k); }
const void* sweep_ptr_stream_u16(int k) { return stream_ptr_for<uint16_t>(k); }
const void* sweep_ptr_stream_u8(int k) { return stream_ptr_for<uint8_t>(k); }
}  // namespace sb
