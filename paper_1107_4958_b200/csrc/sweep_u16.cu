// sweep_u16.cu - instantiations of the sweep kernels for uint16_t sources.
#include "sweep_kernels.cuh"

namespace sb {
const void* sweep_ptr_u16(Mode m, int k) { return sweep_ptr_for<uint16_t>(m, k); }
const void* sweep_ptr_stream_u16(int k) { return stream_ptr_for<uint16_t>(k); }
const void* sweep_ptr_stream_u8(int k) { return stream_ptr_for<uint8_t>(k); }
const void* sweep_ptr_stream_mc_u8(int k) { return stream_mc_ptr_for<uint8_t>(k); }
const void* sweep_ptr_stream_mc_u16(int k) { return stream_mc_ptr_for<uint16_t>(k); }
const void* sweep_ptr_stream_mc_f32(int k);
const void* sweep_ptr_stream_mc_f64(int k);
const void* sweep_ptr_stream_mc(int src_dtype, int k) {
  switch (src_dtype) {
    case SB_DTYPE_U8: return sweep_ptr_stream_mc_u8(k);
    case SB_DTYPE_U16: return sweep_ptr_stream_mc_u16(k);
    case SB_DTYPE_F32: return sweep_ptr_stream_mc_f32(k);
    default: return sweep_ptr_stream_mc_f64(k);
  }
}
const void* sweep_ptr_stream_out_f32(int k);
const void* sweep_ptr_stream_out_f64(int k);
const void* sweep_ptr_stream_out(int src_dtype, int k) {
  switch (src_dtype) {
    case SB_DTYPE_U8: return stream_out_ptr_for<uint8_t>(k);
    case SB_DTYPE_U16: return stream_out_ptr_for<uint16_t>(k);
    case SB_DTYPE_F32: return sweep_ptr_stream_out_f32(k);
    default: return sweep_ptr_stream_out_f64(k);
  }
}
}  // namespace sb
