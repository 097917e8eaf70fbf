// Narrow-band tile refinement on the device: "If a tile
// intersects the zero level set of the signed distance function, its target level is set
// to l0+2.  Otherwise, its target level is set to l0", refined top-down, then repaired to a
// 2:1-graded octree (face-adjacent leaves differ by at most one level).
//
// Every level l0..l0+extra is a dense occupancy bitmap over its (ext << l)^3 tile positions:
// E (the tile exists), R (it is refined: its 8 children exist), M (marked for refinement by
// the grading repair).  Top-down: a level-l tile that exists and intersects the sphere
// surface (the strict box test d_min < r < d_max, reading 16) is refined.  Grading
// repair to fixpoint: every leaf covering a face-neighbour position of a leaf two or more
// levels finer is marked, all marks are refined at once, repeat — each refinement is forced
// in any graded refinement of the current tree, so the fixpoint is the unique minimal graded
// refinement (the same as octgen's host repair and octmg_grade_repair_host).  The leaves
// (E and not R) are emitted as (level, i, j, k).  fp64 geometry compiled with -fmad=false:
// the box test is the IEEE computation the host generator makes, so the tile set is exact.
#include <vector>

#include "octmg_internal.cuh"

namespace octmg {

namespace {

struct BandLevel {
  int nx, ny, nz;
  unsigned* E;
  unsigned* R;
  unsigned* M;
};

struct BandArgs {
  BandLevel lv[OCTMG_MAX_LEVELS];
  int l0, lmax;
  double cx, cy, cz, r;
};

__device__ __forceinline__ bool getb(const unsigned* b, long long i) { return (b[i >> 5] >> (i & 31)) & 1u; }
__device__ __forceinline__ void setb(unsigned* b, long long i) { atomicOr(b + (i >> 5), 1u << (i & 31)); }
__device__ __forceinline__ long long bidx(const BandLevel& L, int i, int j, int k) {
  return ((long long)k * L.ny + j) * L.nx + i;
}

// strict box-vs-sphere-surface test of tile (l, i, j, k): d_min < r < d_max
__device__ bool box_hits_surface(const BandArgs& A, int l, int i, int j, int k) {
  const double size = ldexp(1.0, -l);
  const double lo[3] = {i * size, j * size, k * size};
  const double c[3] = {A.cx, A.cy, A.cz};
  double dmin2 = 0.0, dmax2 = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double hi = lo[a] + size;
    const double nearest = fmin(fmax(c[a], lo[a]), hi);
    const double dn = nearest - c[a];
    dmin2 = dmin2 + dn * dn;
    const double far = fmax(fabs(c[a] - lo[a]), fabs(c[a] - hi));
    dmax2 = dmax2 + far * far;
  }
  const double dmin = sqrt(dmin2), dmax = sqrt(dmax2);
  return dmin < A.r && A.r < dmax;
}

__device__ void refine(const BandArgs& A, int l, int i, int j, int k) {
  setb(A.lv[l].R, bidx(A.lv[l], i, j, k));
  const BandLevel& C = A.lv[l + 1];
  for (int d = 0; d < 8; ++d) setb(C.E, bidx(C, 2 * i + (d & 1), 2 * j + ((d >> 1) & 1), 2 * k + (d >> 2)));
}

// top-down: the existing tiles of level l that intersect the surface are refined
__global__ void k_band_level(BandArgs A, int l) {
  const BandLevel& L = A.lv[l];
  const long long n = (long long)L.nx * L.ny * L.nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (l > A.l0 && !getb(L.E, p)) continue;
    const int i = (int)(p % L.nx), j = (int)((p / L.nx) % L.ny), k = (int)(p / ((long long)L.nx * L.ny));
    if (l == A.l0) setb(L.E, p);
    if (l < A.lmax && box_hits_surface(A, l, i, j, k)) refine(A, l, i, j, k);
  }
}

// grading: mark every leaf covering a face-neighbour position of a leaf of level l two or
// more levels finer
__global__ void k_grade_mark(BandArgs A, int l, int* flag) {
  const BandLevel& L = A.lv[l];
  const long long n = (long long)L.nx * L.ny * L.nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (!getb(L.E, p) || getb(L.R, p)) continue;  // leaves only
    const int i = (int)(p % L.nx), j = (int)((p / L.nx) % L.ny), k = (int)(p / ((long long)L.nx * L.ny));
    for (int f = 0; f < 6; ++f) {
      int q[3] = {i, j, k};
      q[f >> 1] += (f & 1) ? 1 : -1;
      if (q[0] < 0 || q[1] < 0 || q[2] < 0 || q[0] >= L.nx || q[1] >= L.ny || q[2] >= L.nz) continue;
      for (int m = A.l0; m <= l - 2; ++m) {  // the leaf covering q, from the coarsest level down
        const BandLevel& Mv = A.lv[m];
        const long long pm = bidx(Mv, q[0] >> (l - m), q[1] >> (l - m), q[2] >> (l - m));
        if (!getb(Mv.E, pm)) break;
        if (!getb(Mv.R, pm)) {
          setb(Mv.M, pm);
          *flag = 1;
          break;
        }
      }
    }
  }
}

__global__ void k_grade_apply(BandArgs A, int m) {
  const BandLevel& L = A.lv[m];
  const long long n = (long long)L.nx * L.ny * L.nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (!getb(L.M, p)) continue;
    const int i = (int)(p % L.nx), j = (int)((p / L.nx) % L.ny), k = (int)(p / ((long long)L.nx * L.ny));
    refine(A, m, i, j, k);
  }
}

__global__ void k_emit_leaves(BandArgs A, int l, octmg_tile* out, unsigned long long* count, long long cap) {
  const BandLevel& L = A.lv[l];
  const long long n = (long long)L.nx * L.ny * L.nz;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    if (!getb(L.E, p) || getb(L.R, p)) continue;
    const unsigned long long o = atomicAdd(count, 1ull);
    if ((long long)o < cap) {
      const int i = (int)(p % L.nx), j = (int)((p / L.nx) % L.ny), k = (int)(p / ((long long)L.nx * L.ny));
      out[o] = octmg_tile{l, i, j, k};
    }
  }
}

}  // namespace

octmg_status band_tiles(const int32_t* ext, int l0, int extra, const double* centre, double radius, int repair,
                        octmg_tile* out_host, int64_t cap, int64_t* n_out, cudaStream_t s) {
  if (!ext || !centre || !n_out || l0 < 0 || extra < 0 || l0 + extra > MAXL || ext[0] < 1 || ext[1] < 1 ||
      ext[2] < 1 || (((int64_t)ext[0] << (l0 + extra)) > (1 << 19))) {
    set_error("octmg_band_tiles: bad argument");
    return OCTMG_E_INVALID;
  }
  BandArgs A{};
  A.l0 = l0;
  A.lmax = l0 + extra;
  A.cx = centre[0];
  A.cy = centre[1];
  A.cz = centre[2];
  A.r = radius;
  std::vector<void*> mem;
  auto cleanup = [&]() {
    for (void* p : mem) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
  };
  for (int l = l0; l <= A.lmax; ++l) {
    BandLevel& L = A.lv[l];
    L.nx = ext[0] << l;
    L.ny = ext[1] << l;
    L.nz = ext[2] << l;
    const size_t words = ((size_t)L.nx * L.ny * L.nz + 31) / 32;
    for (unsigned** b : {&L.E, &L.R, &L.M}) {
      void* p = nullptr;
      if (cudaMallocAsync(&p, words * 4, s) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        set_error("device allocation failed (band refinement)");
        return OCTMG_E_OOM;
      }
      mem.push_back(p);
      *b = (unsigned*)p;
      OCTMG_CUDA(cudaMemsetAsync(p, 0, words * 4, s));
    }
  }
  auto grid_of = [](const BandLevel& L) {
    const long long n = (long long)L.nx * L.ny * L.nz;
    return (int)std::min<long long>((n + 255) / 256, 148 * 32);
  };
  for (int l = l0; l <= A.lmax; ++l) k_band_level<<<grid_of(A.lv[l]), 256, 0, s>>>(A, l);
  int* dflag = nullptr;
  unsigned long long* dcount = nullptr;
  OCTMG_CUDA(cudaMallocAsync(&dflag, sizeof(int) + sizeof(unsigned long long) * 2, s));
  mem.push_back(dflag);
  dcount = reinterpret_cast<unsigned long long*>(dflag + 2);
  for (int it = 0; repair && it < 64; ++it) {  // each round refines >= 1 tile; depth-bounded in practice
    OCTMG_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), s));
    for (int l = l0 + 2; l <= A.lmax; ++l) k_grade_mark<<<grid_of(A.lv[l]), 256, 0, s>>>(A, l, dflag);
    int flag = 0;
    OCTMG_CUDA(cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
    OCTMG_CUDA(cudaStreamSynchronize(s));
    if (!flag) break;
    for (int m = l0; m <= A.lmax - 2; ++m) {
      k_grade_apply<<<grid_of(A.lv[m]), 256, 0, s>>>(A, m);
      const size_t words = ((size_t)A.lv[m].nx * A.lv[m].ny * A.lv[m].nz + 31) / 32;
      OCTMG_CUDA(cudaMemsetAsync(A.lv[m].M, 0, words * 4, s));
    }
  }
  // the leaves
  octmg_tile* dout = nullptr;
  const int64_t dcap = std::max<int64_t>(cap, 1);
  OCTMG_CUDA(cudaMallocAsync(&dout, sizeof(octmg_tile) * dcap, s));
  mem.push_back(dout);
  OCTMG_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), s));
  for (int l = l0; l <= A.lmax; ++l) k_emit_leaves<<<grid_of(A.lv[l]), 256, 0, s>>>(A, l, dout, dcount, cap);
  OCTMG_CUDA(cudaGetLastError());
  unsigned long long n = 0;
  OCTMG_CUDA(cudaMemcpyAsync(&n, dcount, sizeof(n), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  *n_out = (int64_t)n;
  if (out_host && cap > 0)
    OCTMG_CUDA(cudaMemcpyAsync(out_host, dout, sizeof(octmg_tile) * std::min<int64_t>(n, cap), cudaMemcpyDeviceToHost, s));
  cleanup();
  OCTMG_CUDA(cudaGetLastError());
  if (out_host && (int64_t)n > cap) {
    set_error("octmg_band_tiles: output capacity too small (n_out holds the count)");
    return OCTMG_E_INVALID;
  }
  return OCTMG_OK;
}

}  // namespace octmg
