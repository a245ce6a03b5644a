// Explicit kernel variants for double data (see efft_registry.cuh).
#include "efft_registry.cuh"

namespace efft {

#define D2(r) case r: *out = make_info<double, PT<double, r, true>, NoTile>(); return true;
#define D3(r) case r: *out = make_info<double, T3<double, r, true>, NoTile>(); return true;
#define D5(r) case r: *out = make_info<double, T5<double, r, true>, NoTile>(); return true;
#define D7(r) case r: *out = make_info<double, T7<double, r, true>, NoTile>(); return true;
bool get_direct_kernel_f64(int rho, KernelInfo* out) {
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

// register-path staged variants (persistent pass_kernel, no TMA)
#define SR(rb) case rb: *out = make_info<double, Tile<double, RA, tile_points(RA) / RA, 256, false, CT<double>::VEC>, PT<double, rb, false>>(); return true;
template <int RA>
static bool staged_reg_f64(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SR(2) SR(4) SR(8) SR(16) SR(32) SR(64) SR(128) SR(256) SR(512)
    default: return false;
  }
}
#undef SR

// complex128 staged passes use the register-path persistent kernel (the
// faster measured generic variant); the large sizes go to lean.cu instead
bool get_staged_kernel_f64(int rho_a, int rho_b, KernelInfo* out) {
  if (rho_a == 256) return staged_reg_f64<256>(rho_b, out);
  if (rho_a == 384) return staged_reg_f64<384>(rho_b, out);
  if (rho_a == 320) return staged_reg_f64<320>(rho_b, out);
  if (rho_a == 448) return staged_reg_f64<448>(rho_b, out);
  return false;
}
}  // namespace efft
