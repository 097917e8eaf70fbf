// Cut-cell geometry of the static tank scene on the GPU: per leaf cell the
// ghost-fluid kind, the six fluid face fractions and the right-hand side, from a signed
// distance function sampled at cell corners (tank scene P:L1605-1616; marching
// squares and the saddle rule as SPEC S:L121-138 states them).  fp64 arithmetic, compiled
// with -fmad=false so that every kind decision (phi < 0) and fraction is the same IEEE
// computation as the fp64 oracle's; fractions are stored as fp32.
#include "octmg_internal.cuh"

namespace octmg {

namespace {

struct TankArgs {
  const int4* tile;     // the tiles the fields cover (leaf tiles, or the inner tiles)
  int NL;
  double ext[3];
  double c[3];
  double r;
  uint8_t* kind;
  float* frac;  // [6][N]
  float* b;
  int64_t N;
};

__device__ double sphere_phi(const double p[3], const double c[3], double r) {
  const double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
  return sqrt(dx * dx + dy * dy + dz * dz) - r;
}

// fluid (phi >= 0) fraction of a unit face, corners in cyclic order (0,0),(1,0),(1,1),(0,1)
__device__ double face_fraction(const double phi[4], double phi_centre) {
  const double PX[4] = {0, 1, 1, 0}, PY[4] = {0, 0, 1, 1};
  bool fl[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) fl[k] = phi[k] >= 0.0;
  const bool saddle = fl[0] == fl[2] && fl[1] == fl[3] && fl[0] != fl[1];
  if (saddle && phi_centre < 0.0) {  // solid centre: two separate fluid corner triangles
    double area = 0.0;
    for (int k = 0; k < 4; ++k) {
      if (!fl[k]) continue;
      const int nx = (k + 1) & 3, pv = (k + 3) & 3;
      const double a = phi[k] / (phi[k] - phi[nx]);
      const double bb = phi[k] / (phi[k] - phi[pv]);
      area += 0.5 * a * bb;
    }
    return fmin(1.0, fmax(0.0, area));
  }
  double px[8], py[8];
  int n = 0;
  for (int e = 0; e < 4; ++e) {
    const int a = e, bq = (e + 1) & 3;
    if (fl[a]) { px[n] = PX[a]; py[n] = PY[a]; ++n; }
    if (fl[a] != fl[bq]) {
      const double t = phi[a] / (phi[a] - phi[bq]);
      px[n] = PX[a] + t * (PX[bq] - PX[a]);
      py[n] = PY[a] + t * (PY[bq] - PY[a]);
      ++n;
    }
  }
  double area = 0.0;
  for (int k = 0; k < n; ++k) {
    const int k1 = (k + 1) % n;
    area += px[k] * py[k1] - px[k1] * py[k];
  }
  return fmin(1.0, fmax(0.0, 0.5 * fabs(area)));
}

// one CTA per leaf tile, one thread per cell
__global__ __launch_bounds__(512) void k_tank_fields(TankArgs A) {
  const int t = blockIdx.x;
  const int off = threadIdx.x;
  const int4 tv = A.tile[t];
  const double h = ldexp(1.0, -tv.x) / 8.0;
  const int64_t i = (int64_t)t * TB3 + off;
  const double cen[3] = {((double)(tv.y * 8 + (off & 7)) + 0.5) * h, ((double)(tv.z * 8 + ((off >> 3) & 7)) + 0.5) * h,
                         ((double)(tv.w * 8 + (off >> 6)) + 0.5) * h};
  const bool solid = A.r > 0.0 && sphere_phi(cen, A.c, A.r) < 0.0;
  A.kind[i] = solid ? 2 : 0;  // Neumann (solid) / fluid
  double wy[2] = {0.0, 0.0};
  for (int f = 0; f < 6; ++f) {
    const int a = f >> 1, side = f & 1;
    const int o1 = a == 0 ? 1 : 0, o2 = a == 2 ? 1 : 2;
    double pc[3] = {cen[0], cen[1], cen[2]};
    pc[a] += (side - 0.5) * h;
    double frac = 1.0;
    if (A.r > 0.0) {
      const int U[4] = {-1, 1, 1, -1}, V[4] = {-1, -1, 1, 1};
      double phi[4];
      for (int k = 0; k < 4; ++k) {
        double q[3] = {pc[0], pc[1], pc[2]};
        q[o1] += 0.5 * U[k] * h;
        q[o2] += 0.5 * V[k] * h;
        phi[k] = sphere_phi(q, A.c, A.r);
      }
      frac = face_fraction(phi, sphere_phi(pc, A.c, A.r));
    }
    const bool lo = pc[a] <= 0.0, hi = pc[a] >= A.ext[a];
    if (a == 1) {  // tank: solid bottom, open (Dirichlet) top
      if (lo) frac = 0.0;
      if (hi) frac = 1.0;
    } else if (lo || hi) {
      frac = 0.0;
    }
    const float ff = (float)frac;
    A.frac[(size_t)f * A.N + i] = ff;
    if (a == 1) wy[side] = (double)ff;
  }
  if (A.b) A.b[i] = solid ? 0.0f : (float)(h * h * (wy[1] - wy[0]));
}

}  // namespace

octmg_status tank_fields(const Tree& T, const double* centre, double radius, uint8_t* kind, float* frac, float* b,
                         cudaStream_t s) {
  if (T.NL == 0) return OCTMG_OK;
  TankArgs A;
  A.tile = T.tile;
  A.NL = T.NL;
  for (int k = 0; k < 3; ++k) {
    A.ext[k] = (double)T.ext[k];
    A.c[k] = centre[k];
  }
  A.r = radius;
  A.kind = kind;
  A.frac = frac;
  A.b = b;
  A.N = (int64_t)T.NL * TB3;
  k_tank_fields<<<T.NL, TB3, 0, s>>>(A);
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

// the same scene on the inner tiles (kinds and face fractions of the coarse cells, for the
// GMG comparison mode's grid-assembled coarse operators)
octmg_status tank_fields_inner(const Tree& T, const double* centre, double radius, uint8_t* kind, float* frac,
                               cudaStream_t s) {
  if (T.NI == 0) return OCTMG_OK;
  TankArgs A;
  A.tile = T.tile + T.NL;
  A.NL = T.NI;
  for (int k = 0; k < 3; ++k) {
    A.ext[k] = (double)T.ext[k];
    A.c[k] = centre[k];
  }
  A.r = radius;
  A.kind = kind;
  A.frac = frac;
  A.b = nullptr;
  A.N = (int64_t)T.NI * TB3;
  k_tank_fields<<<T.NI, TB3, 0, s>>>(A);
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

}  // namespace octmg
