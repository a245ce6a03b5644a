// Explicit kernel variants for float data (see efft_registry.cuh).
#include "efft_registry.cuh"

namespace efft {

#define D2(r) case r: *out = make_info<float, PT<float, r, true>, NoTile>(); return true;
#define D3(r) case r: *out = make_info<float, T3<float, r, true>, NoTile>(); return true;
bool get_direct_kernel_f32(int rho, KernelInfo* out) {
  switch (rho) {
    D2(2) D2(4) D2(8) D2(16) D2(32) D2(64) D2(128) D2(256) D2(512)
    D3(3) D3(6) D3(12) D3(24) D3(48) D3(96) D3(192) D3(384)
    default: return false;
  }
}
#undef D2
#undef D3

// complex64 warp-specialised tiles: 8 consumer warps x 32 elements (radix-32
// stages), three TMA buffers in flight
#define SA(rb) case rb: *out = make_info<float, ST<float, RA>, ST<float, rb>, true, false, 3>(); return true;
template <int RA>
static bool staged_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SA(2) SA(4) SA(8) SA(16) SA(32) SA(64) SA(128) SA(256) SA(512)
    default: return false;
  }
}
#undef SA

// register-path staged variants (persistent pass_kernel, no TMA)
#define SR(rb) case rb: *out = make_info<float, Tile<float, RA, (RA % 3 ? 512 : 384) / RA, 256, false, CT<float>::VEC>, PT<float, rb, false>>(); return true;
template <int RA>
static bool staged_reg_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SR(2) SR(4) SR(8) SR(16) SR(32) SR(64) SR(128) SR(256) SR(512)
    default: return false;
  }
}
#undef SR

// 32 KB complex64 tiles: 256 points per column group, 16 elements per thread,
// radix-16 stages, 4 CTAs (32 warps) per SM
template <int RHO> using SM32 = Tile<float, RHO, 256 / RHO, 256, false, 1>;
#define SS(rb) case rb: *out = make_info<float, SM32<256>, SM32<rb>>(); return true;
// 64 KB complex64 tiles with 512 threads (16 elements each, 2 CTAs = 32 warps per SM)
template <int RHO> using W512 = Tile<float, RHO, 512 / RHO, 512, false, 1>;
#define SW(rb) case rb: *out = make_info<float, W512<256>, W512<rb>>(); return true;
#define SP(rb) case rb: *out = make_info<float, W512<256>, W512<rb>, false, true>(); return true;
// software-pipelined (register double-buffered) variant of the same tiles
bool get_staged_pf_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SP(8) SP(16) SP(32) SP(64) SP(128) SP(256)
    default: return false;
  }
}
#undef SP
bool get_staged_wide_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SW(8) SW(16) SW(32) SW(64) SW(128) SW(256)
    default: return false;
  }
}
#undef SW

// warp-specialised 32 KB tiles: 1 producer + 8 consumer warps x 16 elements,
// 3 TMA buffers, 2 CTAs per SM (16 consumer warps per SM)
template <int RHO> using WS32 = Tile<float, RHO, 256 / RHO, 256, false, 1, 32, 1, true>;
#define SW3(rb) case rb: *out = make_info<float, WS32<256>, WS32<rb>, true, false, 3>(); return true;
bool get_staged_ws32_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SW3(8) SW3(16) SW3(32) SW3(64) SW3(128) SW3(256)
    default: return false;
  }
}
#undef SW3

// TMA-prefetching direct tiles (64 KB, 512 threads x 16 elements, 3 buffers)
template <int RHO> using TD = Tile<float, RHO, 512 / RHO, 512, false, 1, 0, 0, true>;
#define DT(r) case r: *out = make_info<float, TD<r>, NoTile, false, false, 3, false, true>(); return true;
bool get_direct_tp_f32(int rho, KernelInfo* out) {
  switch (rho) {
    DT(16) DT(32) DT(64) DT(128) DT(256) DT(512)
    default: return false;
  }
}
#undef DT

// TMA-prefetching tiles: 512 threads x 16 elements, 3 buffers in flight
template <int RHO> using TP16 = Tile<float, RHO, 512 / RHO, 512, false, 1, 0, 0, true>;
#define ST3(rb) case rb: *out = make_info<float, TP16<256>, TP16<rb>, false, false, 3, true>(); return true;
bool get_staged_tp_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    ST3(8) ST3(16) ST3(32) ST3(64) ST3(128) ST3(256)
    default: return false;
  }
}
#undef ST3

bool get_staged_small_f32(int rho_b, KernelInfo* out) {
  switch (rho_b) {
    SS(2) SS(4) SS(8) SS(16) SS(32) SS(64) SS(128) SS(256)
    default: return false;
  }
}
#undef SS

bool get_staged_kernel_f32(int rho_a, int rho_b, int ws, KernelInfo* out) {
  if (ws) {
    if (rho_a == 256) return staged_f32<256>(rho_b, out);
    if (rho_a == 384) return staged_f32<384>(rho_b, out);
  } else {
    if (rho_a == 256) return staged_reg_f32<256>(rho_b, out);
    if (rho_a == 384) return staged_reg_f32<384>(rho_b, out);
  }
  return false;
}

}  // namespace efft
