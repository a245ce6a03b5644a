// Explicit kernel variants for double data (see efft_registry.cuh).
#include "efft_registry.cuh"

namespace efft {

#define D2(r) case r: *out = make_info<double, PT<double, r, true>, NoTile>(); return true;
#define D3(r) case r: *out = make_info<double, T3<double, r, true>, NoTile>(); return true;
bool get_direct_kernel_f64(int rho, KernelInfo* out) {
  switch (rho) {
    D2(2) D2(4) D2(8) D2(16) D2(32) D2(64) D2(128) D2(256) D2(512)
    D3(3) D3(6) D3(12) D3(24) D3(48) D3(96) D3(192) D3(384)
    default: return false;
  }
}
#undef D2
#undef D3

#define SA(rb) case rb: *out = make_info<double, ST<double, RA>, ST<double, rb>, true>(); return true;
template <int RA>
static bool staged_f64(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SA(2) SA(4) SA(8) SA(16) SA(32) SA(64) SA(128) SA(256) SA(512)
    default: return false;
  }
}
#undef SA

// register-path staged variants (persistent pass_kernel, no TMA)
#define SR(rb) case rb: *out = make_info<double, Tile<double, RA, (RA % 3 ? 512 : 384) / RA, 256, false, CT<double>::VEC>, PT<double, rb, false>>(); return true;
template <int RA>
static bool staged_reg_f64(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SR(2) SR(4) SR(8) SR(16) SR(32) SR(64) SR(128) SR(256) SR(512)
    default: return false;
  }
}
#undef SR

// software-pipelined complex128 tiles: 512 threads x 8 elements (64 KB)
template <int RHO> using P512 = Tile<double, RHO, 512 / RHO, 512, false, 1>;
#define SP(rb) case rb: *out = make_info<double, P512<256>, P512<rb>, false, true>(); return true;
bool get_staged_pf_f64(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SP(8) SP(16) SP(32) SP(64) SP(128) SP(256)
    default: return false;
  }
}
#undef SP

// TMA-prefetching complex128 tiles: 256 threads x 16 elements, 3 buffers
template <int RHO> using TP8 = Tile<double, RHO, 512 / RHO, 256, false, 1, 0, 0, true>;
#define ST3(rb) case rb: *out = make_info<double, TP8<256>, TP8<rb>, false, false, 3, true>(); return true;
bool get_staged_tp_f64(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    ST3(8) ST3(16) ST3(32) ST3(64) ST3(128) ST3(256)
    default: return false;
  }
}
#undef ST3

bool get_staged_kernel_f64(int rho_a, int rho_b, int ws, KernelInfo* out) {
  if (ws) {
    if (rho_a == 256) return staged_f64<256>(rho_b, out);
    if (rho_a == 384) return staged_f64<384>(rho_b, out);
  } else {
    if (rho_a == 256) return staged_reg_f64<256>(rho_b, out);
    if (rho_a == 384) return staged_reg_f64<384>(rho_b, out);
  }
  return false;
}

}  // namespace efft
