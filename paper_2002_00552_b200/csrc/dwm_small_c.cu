// dwm_small_c.cu -- dispatch for the fused small-C forward (dwm_small_c.cuh);
// the per-C_in kernels are instantiated in dwm_small_c_c{1..4}.cu so the
// four heavy translation units compile in parallel.
#include "dwm_small_c.cuh"

namespace dwm {
using smallc::Cfg;
using smallc::SMEM_CAP;
using smallc::launch_cc;

bool small_c_supported(const dwm_desc_t& d) {
  if (d.c < 1 || d.c > 4) return false;
  if (d.tiles + 256 >= (int64_t)1 << 31) return false;  // 32-bit tile indexing
  size_t narrow = 0;  // the fallback variant's shared memory (resident U grows with the freqs)
  switch (d.c) {
    case 1: narrow = Cfg<1, 4, 4>::smem_bytes(d.num_freqs); break;
    case 2: narrow = Cfg<2, 4, 4>::smem_bytes(d.num_freqs); break;
    case 3: narrow = Cfg<3, 4, 4>::smem_bytes(d.num_freqs); break;
    default: narrow = Cfg<4, 4, 4>::smem_bytes(d.num_freqs); break;
  }
  return narrow <= SMEM_CAP;
}

int launch_small_c(const dwm_desc_t& d, const void* x, const void* U, void* y, int32_t* flag, cudaStream_t s) {
  const float* xf = (const float*)x;
  const float* Uf = (const float*)U;
  float* yf = (float*)y;
  switch (d.c) {
    case 1: return launch_cc<1>(d, xf, Uf, yf, flag, s);
    case 2: return launch_cc<2>(d, xf, Uf, yf, flag, s);
    case 3: return launch_cc<3>(d, xf, Uf, yf, flag, s);
    case 4: return launch_cc<4>(d, xf, Uf, yf, flag, s);
    default: return fail(DWM_EUNSUPPORTED, "small-C kernel handles C_in <= 4, got %d", d.c);
  }
}

}  // namespace dwm
