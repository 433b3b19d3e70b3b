// Dispatcher of the DMMA TSQR kernels (tsqr_mma_impl.cuh); the instances live in their own
// translation units (tsqr_mma_inst.cu, one per configuration listed in build.py).
#include <cstdlib>

#include "kernels.h"

namespace sqb {

// (8-column tiles, 8-row groups per panel, warps per CTA) - keep in sync with MMA_CONFIGS in build.py
#define SQB_MMA_CONFIGS(X) \
  X(2, 16, 8) X(3, 12, 8) X(4, 10, 8) X(5, 8, 8) X(6, 6, 8) X(7, 6, 8) X(8, 6, 8)

#define SQB_DECL(NBV, RGV, NWV) \
  cudaError_t launch_tsqr_mma_##NBV##_##RGV##_##NWV(const TsqrParams&, long long, cudaStream_t);
SQB_MMA_CONFIGS(SQB_DECL)
#undef SQB_DECL


// column count -> configuration (largest panel the register file holds: w takes 2*NB*RG doubles)
#define SQB_MMA_SWITCH(EXPR)               \
  switch ((n + 7) / 8) {                   \
    case 2: return EXPR(2, 16, 8);         \
    case 3: return EXPR(3, 12, 8);         \
    case 4: return EXPR(4, 10, 8);         \
    case 5: return EXPR(5, 8, 8);          \
    case 6: return EXPR(6, 6, 8);          \
    case 7: return EXPR(7, 6, 8);          \
    default: return EXPR(8, 6, 8);         \
  }

cudaError_t launch_tsqr_mma(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int n = prm.n;
  if (n < kMmaTsqrMinN || n > 64) return cudaErrorInvalidValue;
#define LG(NBV, RGV, NWV) launch_tsqr_mma_##NBV##_##RGV##_##NWV(prm, num_blocks, stream)
  SQB_MMA_SWITCH(LG)
#undef LG
}

int tsqr_mma_panel_rows(int n) {
#define CG(NBV, RGV, NWV) (8 * RGV)
  SQB_MMA_SWITCH(CG)
#undef CG
}

int tsqr_mma_warps(int n) {
#define WG(NBV, RGV, NWV) NWV
  SQB_MMA_SWITCH(WG)
#undef WG
}

}  // namespace sqb
