// mm_i32.cu -- LUT-MM kernel instantiations for the REPR_I32 table representation.
#include "mm_launch.cuh"

namespace axq {
int launch_mm_i32(int epi, int loader, const MMArgs& p, const Cfg& c, dim3 grid, cudaStream_t st) {
    return launch_mm_repr<REPR_I32>(epi, loader, p, c, grid, st);
}
}  // namespace axq
