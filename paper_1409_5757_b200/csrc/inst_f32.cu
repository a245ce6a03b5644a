// Explicit kernel variants for float data (see efft_registry.cuh).
#include "efft_registry.cuh"

namespace efft {

#define D2(r) case r: *out = make_info<float, PT<float, r, true>, NoTile>(); return true;
#define D3(r) case r: *out = make_info<float, T3<float, r, true>, NoTile>(); return true;
#define D5(r) case r: *out = make_info<float, T5<float, r, true>, NoTile>(); return true;
#define D7(r) case r: *out = make_info<float, T7<float, r, true>, NoTile>(); return true;
bool get_direct_kernel_f32(int rho, KernelInfo* out) {
  switch (rho) {
    D2(2) D2(4) D2(8) D2(16) D2(32) D2(64) D2(128) D2(256) D2(512)
    D3(3) D3(6) D3(12) D3(24) D3(48) D3(96) D3(192) D3(384)
    D5(5) D5(10) D5(20) D5(40) D5(80) D5(160) D5(320)
    D7(7) D7(14) D7(28) D7(56) D7(112) D7(224) D7(448)
    default: return false;
  }
}
#undef D2
#undef D3
#undef D5
#undef D7

// complex64 warp-specialised tiles: 8 consumer warps x 32 elements (radix-32
// stages), three TMA buffers in flight
#define SA(rb) case rb: *out = make_info<float, ST<float, RA>, ST<float, rb>, true, 3>(); return true;
template <int RA>
static bool staged_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SA(2) SA(4) SA(8) SA(16) SA(32) SA(64) SA(128) SA(256) SA(512)
    default: return false;
  }
}
#undef SA

// complex64 staged passes use the warp-specialised TMA kernel (the faster
// measured generic variant); the large sizes go to lean.cu instead
bool get_staged_kernel_f32(int rho_a, int rho_b, KernelInfo* out) {
  if (rho_a == 256) return staged_f32<256>(rho_b, out);
  if (rho_a == 384) return staged_f32<384>(rho_b, out);
  if (rho_a == 320) return staged_f32<320>(rho_b, out);
  if (rho_a == 448) return staged_f32<448>(rho_b, out);
  return false;
}

}  // namespace efft
