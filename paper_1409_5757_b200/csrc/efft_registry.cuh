// efft_registry.cuh -- compiled tile/kernel variants the planner can pick from.
#pragma once
#include "efft_kernels.cuh"

namespace efft {

struct KernelInfo {
  void (*fn)(PassArgs);
  int nt;          // threads per CTA
  int smem_bytes;  // dynamic shared memory
  int rho_a, d_a, e_a;
  int rho_b, d_b, e_b;
  int stages_a[12], nst_a;
  int stages_b[12], nst_b;
  int ws;    // warp-specialised TMA kernel (needs tensor maps)
  int tpts;    // D * RHO of the A tiles (points per column group per task)
  int tpts_b;  // D * RHO of the B tiles
};

// Power-of-two tiles hold D*RHO = 512 points per column group, radix-3 tiles
// 384, radix-5 tiles 320 and radix-7 tiles 448 (one complex element per lane
// access: EV = 10..28 takes radix-20/14/10/7/5 stages); 256 threads; F columns
// of 128 bytes.
template <typename R, int RHO, bool MASK> using PT = Tile<R, RHO, 512 / RHO, 256, MASK, CT<R>::VEC>;
template <typename R, int RHO, bool MASK> using T3 = Tile<R, RHO, 384 / RHO, 256, MASK, CT<R>::VEC>;
template <typename R, int RHO, bool MASK> using T5 = Tile<R, RHO, 320 / RHO, 256, MASK, 1>;
template <typename R, int RHO, bool MASK> using T7 = Tile<R, RHO, 448 / RHO, 256, MASK, 1>;
// points per column group of a tile whose radix is RHO
constexpr int tile_points(int rho) {
  return rho % 3 == 0 ? 384 : rho % 5 == 0 ? 320 : rho % 7 == 0 ? 448 : 512;
}
// Consumer tiles of the warp-specialised staged kernel: 256 consumer threads
// after the producer warp (TOFF 32), named barrier 1, one complex element per
// lane access.
template <typename R, int RHO> using ST = Tile<R, RHO, tile_points(RHO) / RHO, 256, false, 1, 32, 1, true>;

template <typename R, class TA, class TB, bool WS = false, int NBUF = 2>
KernelInfo make_info() {
  using V = typename CT<R>::V;
  KernelInfo k{};
  const int sm = TA::SMEM_ELEMS > TB::SMEM_ELEMS ? TA::SMEM_ELEMS : TB::SMEM_ELEMS;
  if constexpr (WS) {
    k.fn = staged_kernel<R, TA, TB, NBUF>;
    k.nt = TA::NT + 32;
    k.smem_bytes = (int)((NBUF * sm + TA::RHO + TB::RHO) * sizeof(V)) + 1024;  // + swizzle alignment slack
    k.ws = 1;
  } else {
    k.fn = pass_kernel<R, TA, TB>;
    k.nt = TA::NT;
    k.smem_bytes = (int)((sm + TA::RHO + TB::RHO) * sizeof(V));
  }
  k.rho_a = TA::RHO;
  k.d_a = TA::D;
  k.tpts = TA::D * TA::RHO;
  k.e_a = TA::E;
  k.nst_a = TA::NST;
  for (int i = 0; i < TA::NST; ++i) k.stages_a[i] = TA::PL.sig[i];
  if constexpr (TB::RHO > 0) {
    k.rho_b = TB::RHO;
    k.tpts_b = TB::D * TB::RHO;
    k.d_b = TB::D;
    k.e_b = TB::E;
    k.nst_b = TB::NST;
    for (int i = 0; i < TB::NST; ++i) k.stages_b[i] = TB::PL.sig[i];
  }
  return k;
}

// Defined in inst_f32.cu / inst_f64.cu.
bool get_direct_kernel_f32(int rho, KernelInfo* out);
bool get_direct_kernel_f64(int rho, KernelInfo* out);
bool get_staged_kernel_f32(int rho_a, int rho_b, KernelInfo* out);
bool get_staged_kernel_f64(int rho_a, int rho_b, KernelInfo* out);

}  // namespace efft
