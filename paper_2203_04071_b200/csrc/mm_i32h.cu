// mm_i32h.cu -- LUT-MM kernel instantiations for the REPR_I32H table representation (SM-resident int32 halves).
#include "mm_launch.cuh"

namespace axq {
int launch_mm_i32h(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st) {
    return launch_mm_repr<REPR_I32H>(epi, loader, p, c, grid, st);
}
}  // namespace axq
