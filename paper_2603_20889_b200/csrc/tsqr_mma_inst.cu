// One (tiles, row groups, warps) instance of the DMMA TSQR kernel per translation unit: with several
// instances in one file nvcc's unroll budget runs out and the register panel is demoted to local
// memory (3.5x slower).  Compiled once per entry of MMA_CONFIGS in build.py with
// -DSQB_MMA_NB=.. -DSQB_MMA_RG=.. -DSQB_MMA_NW=..
#include "tsqr_mma_impl.cuh"

#define SQB_CAT_(a, b, c, d) a##_##b##_##c##_##d
#define SQB_CAT(a, b, c, d) SQB_CAT_(a, b, c, d)

namespace sqb {

cudaError_t SQB_CAT(launch_tsqr_mma, SQB_MMA_NB, SQB_MMA_RG, SQB_MMA_NW)(const TsqrParams& prm, long long num_blocks,
                                                                       cudaStream_t stream) {
  return launch_cfg<SQB_MMA_NB, SQB_MMA_RG, SQB_MMA_NW>(prm, num_blocks, stream);
}

}  // namespace sqb
