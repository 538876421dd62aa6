// BEM element integrals on the device (reading R-BEM).
// Sources are flat triangles with piecewise-constant densities; collocation points are
// the centroids.  int_T G(x, y) dy with G = 1/(4 pi |x - y|):
//   self (x = the element's own collocation point): analytic flat-triangle value
//        sum over edges of h_e ln((s2 + r2) / (s1 + r1)), / 4 pi;
//   |x - centroid| > 2 diam (longest edge): Dunavant's 6-point degree-4 rule;
//   otherwise: 4-way midpoint subdivision, recursively (explicit stack), the rule at depth 8.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace kifmm {

struct DTri {
  double v[3][3];
};

__device__ __forceinline__ DTri load_tri(const double4* t3) {  // 3 x double4 (x, y, z, pad)
  DTri T;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const double4 a = t3[e];
    T.v[e][0] = a.x; T.v[e][1] = a.y; T.v[e][2] = a.z;
  }
  return T;
}

__device__ __forceinline__ double tri_area_d(const DTri& T) {
  const double a0 = T.v[1][0] - T.v[0][0], a1 = T.v[1][1] - T.v[0][1], a2 = T.v[1][2] - T.v[0][2];
  const double b0 = T.v[2][0] - T.v[0][0], b1 = T.v[2][1] - T.v[0][1], b2 = T.v[2][2] - T.v[0][2];
  const double c0 = a1 * b2 - a2 * b1, c1 = a2 * b0 - a0 * b2, c2 = a0 * b1 - a1 * b0;
  return 0.5 * sqrt(c0 * c0 + c1 * c1 + c2 * c2);
}

__device__ __forceinline__ double tri_diam_d(const DTri& T) {
  double m = 0;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const int f = e == 2 ? 0 : e + 1;
    const double dx = T.v[e][0] - T.v[f][0], dy = T.v[e][1] - T.v[f][1], dz = T.v[e][2] - T.v[f][2];
    m = fmax(m, sqrt(dx * dx + dy * dy + dz * dz));
  }
  return m;
}

__device__ __forceinline__ double tri_rule6_d(const DTri& T, const double x[3]) {
  const double A[2] = {0.445948490915965, 0.091576213509771};
  const double W[2] = {0.223381589678011, 0.109951743655322};
  double acc = 0;
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int perm = 0; perm < 3; ++perm) {
      double l0 = A[g], l1 = A[g], l2 = A[g];
      if (perm == 0) l0 = 1.0 - 2.0 * A[g];
      if (perm == 1) l1 = 1.0 - 2.0 * A[g];
      if (perm == 2) l2 = 1.0 - 2.0 * A[g];
      const double y0 = l0 * T.v[0][0] + l1 * T.v[1][0] + l2 * T.v[2][0];
      const double y1 = l0 * T.v[0][1] + l1 * T.v[1][1] + l2 * T.v[2][1];
      const double y2 = l0 * T.v[0][2] + l1 * T.v[1][2] + l2 * T.v[2][2];
      const double dx = x[0] - y0, dy = x[1] - y1, dz = x[2] - y2;
      acc += W[g] / sqrt(dx * dx + dy * dy + dz * dz);
    }
  return acc * tri_area_d(T) * kInv4Pi;
}

__device__ __forceinline__ double tri_self_d(const DTri& T, const double x[3]) {
  double acc = 0;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const int f = e == 2 ? 0 : e + 1;
    double t0 = T.v[f][0] - T.v[e][0], t1 = T.v[f][1] - T.v[e][1], t2 = T.v[f][2] - T.v[e][2];
    const double L = sqrt(t0 * t0 + t1 * t1 + t2 * t2);
    t0 /= L; t1 /= L; t2 /= L;
    const double p0 = T.v[e][0] - x[0], p1 = T.v[e][1] - x[1], p2 = T.v[e][2] - x[2];
    const double q0 = T.v[f][0] - x[0], q1 = T.v[f][1] - x[1], q2 = T.v[f][2] - x[2];
    const double s1 = p0 * t0 + p1 * t1 + p2 * t2, s2 = q0 * t0 + q1 * t1 + q2 * t2;
    const double r1 = sqrt(p0 * p0 + p1 * p1 + p2 * p2), r2 = sqrt(q0 * q0 + q1 * q1 + q2 * q2);
    const double h = sqrt(fmax(0.0, r1 * r1 - s1 * s1));
    acc += h * log((s2 + r2) / (s1 + r1));
  }
  return acc * kInv4Pi;
}

__device__ __forceinline__ bool tri_regular(const DTri& T, const double x[3]) {
  const double c0 = (T.v[0][0] + T.v[1][0] + T.v[2][0]) / 3.0;
  const double c1 = (T.v[0][1] + T.v[1][1] + T.v[2][1]) / 3.0;
  const double c2 = (T.v[0][2] + T.v[1][2] + T.v[2][2]) / 3.0;
  const double dx = x[0] - c0, dy = x[1] - c1, dz = x[2] - c2;
  return sqrt(dx * dx + dy * dy + dz * dz) > 2.0 * tri_diam_d(T);
}

// int_T G(x, y) dy; self: x is T's own collocation point (analytic)
static __device__ __noinline__ double bem_integral(const DTri& T0, const double x[3], bool self) {
  if (self) return tri_self_d(T0, x);
  if (tri_regular(T0, x)) return tri_rule6_d(T0, x);
  constexpr int kMaxDepth = 8, kStack = 3 * kMaxDepth + 2;
  DTri st[kStack];
  int dep[kStack];
  int sp = 0;
  st[0] = T0;
  dep[0] = 0;
  sp = 1;
  double acc = 0;
  while (sp > 0) {
    --sp;
    const DTri T = st[sp];
    const int d = dep[sp];
    if (d >= kMaxDepth || tri_regular(T, x)) {
      acc += tri_rule6_d(T, x);
      continue;
    }
    double m[3][3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      const int f = e == 2 ? 0 : e + 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) m[e][c] = 0.5 * (T.v[e][c] + T.v[f][c]);
    }
    // children: (v0, m01, m20), (m01, v1, m12), (m20, m12, v2), (m01, m12, m20)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      st[sp].v[0][c] = T.v[0][c]; st[sp].v[1][c] = m[0][c]; st[sp].v[2][c] = m[2][c];
      st[sp + 1].v[0][c] = m[0][c]; st[sp + 1].v[1][c] = T.v[1][c]; st[sp + 1].v[2][c] = m[1][c];
      st[sp + 2].v[0][c] = m[2][c]; st[sp + 2].v[1][c] = m[1][c]; st[sp + 2].v[2][c] = T.v[2][c];
      st[sp + 3].v[0][c] = m[0][c]; st[sp + 3].v[1][c] = m[1][c]; st[sp + 3].v[2][c] = m[2][c];
    }
    dep[sp] = dep[sp + 1] = dep[sp + 2] = dep[sp + 3] = d + 1;
    sp += 4;
  }
  return acc;
}

}  // namespace kifmm
