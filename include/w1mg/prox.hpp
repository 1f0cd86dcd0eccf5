// prox.hpp -- pointwise proximal maps (host scalars).  Source-compatible with
// /root/reference/proj/include/w1mg/prox.hpp; the device twins used inside
// the fused kernels live in paper_1810_00118_b200/csrc/device_common.cuh.
#pragma once

#include "w1mg/pnorm.hpp"

namespace w1mg {

/// argmin_u ||u||_p + ||u - v||^2 / (2 mu); mu > 0.
Vec2 shrink(Vec2 v, double mu, PNorm p);
/// Nearest point of the unit q-ball.
Vec2 project_unit_ball(Vec2 v, PNorm q);
/// Nearest point of {u : ||u||_1 <= radius}; radius > 0.
Vec2 project_l1_ball(Vec2 v, double radius);

}  // namespace w1mg
