// wide_pk_geo.h -- host-visible constants of the packed wide LUT-GEMM (wide_pk.cuh).
#pragma once

namespace axq {
namespace wpk {
constexpr int KP_ALIGN = 8;   // Kp: a multiple of every stage depth KS and of the 8-code A loads
}  // namespace wpk
}  // namespace axq
