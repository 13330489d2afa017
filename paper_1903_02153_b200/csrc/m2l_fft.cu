// Uniform-grid M2L (engine.py:258-292) — placeholder until the FFT-diagonal
// Hadamard kernel lands; the host refuses the uniform scheme loudly.
#include "common.cuh"

using namespace bfmm;

extern "C" int bfmm_m2l_fft_scratch_bytes(int level, int m, int p,
                                          size_t *bytes) {
  (void)level; (void)m; (void)p;
  *bytes = 0;
  set_error("bfmm_m2l_fft: not implemented in this build");
  return 5;
}

extern "C" int bfmm_m2l_fft(const double *moments, double *locals, int level,
                            int m, int p, const double *symbols, double scale,
                            void *scratch, size_t scratch_bytes,
                            bfmm_stream_t stream) {
  (void)moments; (void)locals; (void)level; (void)m; (void)p; (void)symbols;
  (void)scale; (void)scratch; (void)scratch_bytes; (void)stream;
  set_error("bfmm_m2l_fft: not implemented in this build");
  return 5;
}
