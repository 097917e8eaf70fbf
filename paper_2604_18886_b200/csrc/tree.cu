// GPU octree construction (P:L548-550 leaf/inner/ghost tiles; P:L893-894 cached
// same-level neighbours).  Keys are (MAXL - level) << 58 | morton(i, j, k) so that one
// ascending radix sort yields the canonical order (level descending, Morton ascending).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "octmg_internal.cuh"

namespace octmg {

namespace {

enum { ERR_INVALID = 1, ERR_OVERLAP = 2, ERR_NOT_GRADED = 4 };

__device__ __forceinline__ uint64_t spread19(uint32_t v) {
  uint64_t x = v & 0x7FFFFu;
  x = (x | (x << 32)) & 0x1F00000000FFFFull;
  x = (x | (x << 16)) & 0x1F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint32_t compact19(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10C30C30C30C30C3ull;
  x = (x ^ (x >> 4)) & 0x100F00F00F00F00Full;
  x = (x ^ (x >> 8)) & 0x1F0000FF0000FFull;
  x = (x ^ (x >> 16)) & 0x1F00000000FFFFull;
  x = (x ^ (x >> 32)) & 0x7FFFFull;
  return (uint32_t)x;
}

__device__ __forceinline__ uint64_t make_key(int l, int i, int j, int k) {
  return ((uint64_t)(MAXL - l) << KEY_LEVEL_SHIFT) | spread19(i) | (spread19(j) << 1) | (spread19(k) << 2);
}

__device__ __forceinline__ int key_level(uint64_t key) { return MAXL - (int)(key >> KEY_LEVEL_SHIFT); }

__device__ __forceinline__ int4 decode_key(uint64_t key) {
  uint64_t m = key & ((1ull << KEY_LEVEL_SHIFT) - 1);
  return make_int4(key_level(key), (int)compact19(m), (int)compact19(m >> 1), (int)compact19(m >> 2));
}

__device__ __forceinline__ int bsearch_key(const uint64_t* keys, int n, uint64_t k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? lo : -1;
}

struct Ext { int e[3]; };

__global__ void k_keys(const int4* in, int64_t n, Ext ext, uint64_t* keys, int* err) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int4 v = in[t];
  bool ok = v.x >= 0 && v.x <= MAXL;
  if (ok) {
    int64_t lim0 = (int64_t)ext.e[0] << v.x, lim1 = (int64_t)ext.e[1] << v.x, lim2 = (int64_t)ext.e[2] << v.x;
    ok = v.y >= 0 && v.z >= 0 && v.w >= 0 && v.y < lim0 && v.z < lim1 && v.w < lim2 &&
         lim0 <= (1 << 19) && lim1 <= (1 << 19) && lim2 <= (1 << 19);
  }
  if (!ok) { atomicOr(err, ERR_INVALID); keys[t] = 0; return; }
  keys[t] = make_key(v.x, v.y, v.z, v.w);
}

__global__ void k_dups(const uint64_t* keys, int n, int* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 1 && t < n && keys[t] == keys[t - 1]) atomicOr(err, ERR_OVERLAP);
}

__global__ void k_anc_count(const uint64_t* keys, int n, int* cnt) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) cnt[t] = key_level(keys[t]);
}

__global__ void k_anc_emit(const uint64_t* keys, int n, const int* off, uint64_t* anc) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int4 v = decode_key(keys[t]);
  int o = off[t];
  int i = v.y, j = v.z, k = v.w;
  for (int m = v.x - 1; m >= 0; --m) {
    i >>= 1; j >>= 1; k >>= 1;
    anc[o++] = make_key(m, i, j, k);
  }
}

__global__ void k_overlap(const uint64_t* leaf, int nl, const uint64_t* inner, int ni, int* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nl && bsearch_key(inner, ni, leaf[t]) >= 0) atomicOr(err, ERR_OVERLAP);
}

__global__ void k_volume(const uint64_t* leaf, int nl, int L, unsigned long long* vol) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (t < nl) v = 1ull << (3 * (L - key_level(leaf[t])));
  // warp pre-reduction
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(vol, v);
}

__global__ void k_level_counts(const uint64_t* keys, int n, int* cnt) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) atomicAdd(&cnt[key_level(keys[t])], 1);
}

__global__ void k_decode(const uint64_t* keys, int n, int4* tile) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) tile[t] = decode_key(keys[t]);
}

__device__ __forceinline__ int find_tile(const uint64_t* lk, int nl, const uint64_t* ik, int ni, int l, int i,
                                         int j, int k) {
  uint64_t key = make_key(l, i, j, k);
  int a = bsearch_key(lk, nl, key);
  if (a >= 0) return a;
  a = bsearch_key(ik, ni, key);
  return a >= 0 ? nl + a : -1;
}

__global__ void k_tables(const int4* tile, const uint64_t* lk, int nl, const uint64_t* ik, int ni, Ext ext,
                         int* nbr, int* parent, int* child, int* gflag, int* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl + ni) return;
  int4 v = tile[t];
  int l = v.x;
  for (int f = 0; f < 6; ++f) {
    int a = f >> 1, s = (f & 1) ? 1 : -1;
    int q[3] = {v.y, v.z, v.w};
    q[a] += s;
    int res;
    if (q[a] < 0 || q[a] >= (ext.e[a] << l)) {
      res = -1;
    } else {
      int n = find_tile(lk, nl, ik, ni, l, q[0], q[1], q[2]);
      if (n >= 0) {
        res = n;
      } else {
        int c = (t < nl && l >= 1) ? bsearch_key(lk, nl, make_key(l - 1, q[0] >> 1, q[1] >> 1, q[2] >> 1)) : -1;
        if (c < 0) { atomicOr(err, ERR_NOT_GRADED); res = -1; }
        else res = -2 - c;
      }
    }
    nbr[6 * t + f] = res;
    if (t < nl && (f & 1)) gflag[3 * t + a] = res <= -2 ? 1 : 0;
  }
  parent[t] = l >= 1 ? nl + bsearch_key(ik, ni, make_key(l - 1, v.y >> 1, v.z >> 1, v.w >> 1)) : -1;
  if (t >= nl) {
    for (int d = 0; d < 8; ++d)
      child[8 * (t - nl) + d] = find_tile(lk, nl, ik, ni, l + 1, 2 * v.y + (d & 1), 2 * v.z + ((d >> 1) & 1),
                                          2 * v.w + (d >> 2));
  }
}

__global__ void k_glayer(const int* gflag, const int* gscan, int n, int* glayer) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) glayer[t] = gflag[t] ? gscan[t] : -1;
}

inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

template <class T>
static octmg_status dalloc(std::vector<void*>& list, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = dev_malloc(count * sizeof(T));
  if (!q) {
    set_error("device allocation failed");
    return OCTMG_E_OOM;
  }
  list.push_back(q);
  *p = (T*)q;
  return OCTMG_OK;
}

Tree::~Tree() {
  if (!allocs.empty()) cudaDeviceSynchronize();  // see Hier::~Hier
  for (void* p : allocs) dev_free(p);
}

octmg_status build_tree(const octmg_tree_desc* desc, const octmg_tile* tiles, int64_t n, cudaStream_t s,
                        Tree* T) {
  if (n <= 0 || n > (1ll << 30)) { set_error("leaf tile count out of range"); return OCTMG_E_INVALID; }
  for (int a = 0; a < 3; ++a) {
    if (desc->ext[a] < 1 || desc->ext[a] > (1 << 10)) { set_error("bad domain extent"); return OCTMG_E_INVALID; }
    T->ext[a] = desc->ext[a];
  }
  for (int f = 0; f < 6; ++f) {
    if (desc->wall_bc[f] > 1) { set_error("wall_bc must be 0 or 1"); return OCTMG_E_INVALID; }
    T->wall[f] = desc->wall_bc[f];
  }
  if (desc->grade_repair != 0) { set_error("grade_repair must be 0 or 1"); return OCTMG_E_INVALID; }  // 1: api.cu repairs first
  if (desc->nranks < 1 || desc->nranks > 64 || desc->rank < 0 || desc->rank >= desc->nranks ||
      (desc->nranks > 1 && !desc->nccl_comm)) {
    set_error("bad rank / nranks / nccl_comm");
    return OCTMG_E_INVALID;
  }
  T->rank = desc->rank;
  T->nranks = desc->nranks;
  T->nccl_comm = desc->nccl_comm;
  std::vector<void*> tmp;  // freed at exit
  struct Guard { std::vector<void*>& v; ~Guard() { for (void* p : v) dev_free(p); } } guard{tmp};
  Ext ext{{T->ext[0], T->ext[1], T->ext[2]}};
  int nl = (int)n;

  int4* d_in; uint64_t *d_k0, *d_k1; int* d_err;
  OCTMG_TRY(dalloc(tmp, &d_in, n));
  OCTMG_TRY(dalloc(tmp, &d_k0, n));
  OCTMG_TRY(dalloc(T->allocs, &T->leaf_keys, n));
  d_k1 = T->leaf_keys;
  OCTMG_TRY(dalloc(tmp, &d_err, 1));
  OCTMG_CUDA(cudaMemcpyAsync(d_in, tiles, n * sizeof(int4), cudaMemcpyHostToDevice, s));
  OCTMG_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  k_keys<<<nblk(n, 256), 256, 0, s>>>(d_in, n, ext, d_k0, d_err);
  size_t tb = 0;
  OCTMG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, d_k0, d_k1, nl, 0, 64, s));
  void* d_tmp;
  size_t tmp_bytes = tb;
  {
    size_t tb2 = 0, tb3 = 0;
    OCTMG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, (int*)nullptr, (int*)nullptr, nl, s));
    tmp_bytes = std::max(tmp_bytes, tb2);
    (void)tb3;
  }
  OCTMG_TRY(dalloc(tmp, (char**)&d_tmp, tmp_bytes));
  OCTMG_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, tb, d_k0, d_k1, nl, 0, 64, s));
  k_dups<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, d_err);
  // inner tiles: all strict ancestors of the leaves
  int* d_cnt; int* d_off;
  OCTMG_TRY(dalloc(tmp, &d_cnt, nl));
  OCTMG_TRY(dalloc(tmp, &d_off, nl));
  k_anc_count<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, d_cnt);
  size_t tb2 = 0;
  OCTMG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, d_cnt, d_off, nl, s));
  OCTMG_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tb2, d_cnt, d_off, nl, s));
  int h_last[2];
  OCTMG_CUDA(cudaMemcpyAsync(&h_last[0], d_off + nl - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(&h_last[1], d_cnt + nl - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  int h_err = 0;
  OCTMG_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  if (h_err & ERR_INVALID) { set_error("leaf tile level or coordinate out of range"); return OCTMG_E_INVALID; }
  if (h_err & ERR_OVERLAP) { set_error("duplicate leaf tiles"); return OCTMG_E_OVERLAP; }
  int64_t n_anc = (int64_t)h_last[0] + h_last[1];
  int ni = 0;
  uint64_t* d_inner = nullptr;
  if (n_anc > 0) {
    uint64_t *d_a0, *d_a1;
    int* d_nsel;
    OCTMG_TRY(dalloc(tmp, &d_a0, n_anc));
    OCTMG_TRY(dalloc(tmp, &d_a1, n_anc));
    OCTMG_TRY(dalloc(tmp, &d_nsel, 1));
    k_anc_emit<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, d_off, d_a0);
    size_t ts = 0, tu = 0;
    OCTMG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, ts, d_a0, d_a1, (int)n_anc, 0, 64, s));
    OCTMG_CUDA(cub::DeviceSelect::Unique(nullptr, tu, d_a1, d_a0, d_nsel, (int)n_anc, s));
    void* d_t2;
    OCTMG_TRY(dalloc(tmp, (char**)&d_t2, std::max(ts, tu)));
    OCTMG_CUDA(cub::DeviceRadixSort::SortKeys(d_t2, ts, d_a0, d_a1, (int)n_anc, 0, 64, s));
    OCTMG_CUDA(cub::DeviceSelect::Unique(d_t2, tu, d_a1, d_a0, d_nsel, (int)n_anc, s));
    OCTMG_CUDA(cudaMemcpyAsync(&ni, d_nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
    OCTMG_CUDA(cudaStreamSynchronize(s));
    OCTMG_TRY(dalloc(T->allocs, &T->inner_keys, ni));
    OCTMG_CUDA(cudaMemcpyAsync(T->inner_keys, d_a0, ni * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
    d_inner = T->inner_keys;
  } else {
    OCTMG_TRY(dalloc(T->allocs, &T->inner_keys, 1));
  }
  if (ni > 0) k_overlap<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, d_inner, ni, d_err);
  // finest level from the first key (finest level sorts first)
  uint64_t k0;
  OCTMG_CUDA(cudaMemcpyAsync(&k0, d_k1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  int L = MAXL - (int)(k0 >> KEY_LEVEL_SHIFT);
  unsigned long long* d_vol;
  OCTMG_TRY(dalloc(tmp, &d_vol, 1));
  OCTMG_CUDA(cudaMemsetAsync(d_vol, 0, sizeof(unsigned long long), s));
  k_volume<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, L, d_vol);
  int* d_lcnt;
  OCTMG_TRY(dalloc(tmp, &d_lcnt, 2 * (MAXL + 1)));
  OCTMG_CUDA(cudaMemsetAsync(d_lcnt, 0, 2 * (MAXL + 1) * sizeof(int), s));
  k_level_counts<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, d_lcnt);
  if (ni) k_level_counts<<<nblk(ni, 256), 256, 0, s>>>(d_inner, ni, d_lcnt + MAXL + 1);
  unsigned long long vol = 0;
  int lcnt[2 * (MAXL + 1)];
  OCTMG_CUDA(cudaMemcpyAsync(&vol, d_vol, sizeof(vol), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(lcnt, d_lcnt, sizeof(lcnt), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  if (h_err & ERR_OVERLAP) { set_error("a leaf tile contains another leaf tile"); return OCTMG_E_OVERLAP; }
  unsigned long long dom = (unsigned long long)T->ext[0] * T->ext[1] * T->ext[2] << (3 * L);
  if (vol != dom) { set_error("leaf tiles do not cover the domain"); return OCTMG_E_GAP; }

  T->L = L;
  T->NL = nl;
  T->NI = ni;
  T->T = nl + ni;
  int acc = 0;
  for (int l = L; l >= 0; --l) { T->lb[l] = acc; T->lc[l] = lcnt[l]; acc += lcnt[l]; }
  acc = nl;
  for (int l = L; l >= 0; --l) { T->ib[l] = acc; T->ic[l] = lcnt[MAXL + 1 + l]; acc += lcnt[MAXL + 1 + l]; }
  for (int l = L + 1; l <= MAXL; ++l) { T->lb[l] = 0; T->lc[l] = 0; T->ib[l] = 0; T->ic[l] = 0; }

  OCTMG_TRY(dalloc(T->allocs, &T->tile, T->T));
  OCTMG_TRY(dalloc(T->allocs, &T->nbr, (size_t)T->T * 6));
  OCTMG_TRY(dalloc(T->allocs, &T->parent, T->T));
  OCTMG_TRY(dalloc(T->allocs, &T->child, (size_t)ni * 8));
  OCTMG_TRY(dalloc(T->allocs, &T->glayer, (size_t)nl * 3));
  int *d_gflag, *d_gscan;
  OCTMG_TRY(dalloc(tmp, &d_gflag, (size_t)nl * 3));
  OCTMG_TRY(dalloc(tmp, &d_gscan, (size_t)nl * 3));
  k_decode<<<nblk(nl, 256), 256, 0, s>>>(d_k1, nl, T->tile);
  if (ni) k_decode<<<nblk(ni, 256), 256, 0, s>>>(d_inner, ni, T->tile + nl);
  k_tables<<<nblk(T->T, 128), 128, 0, s>>>(T->tile, d_k1, nl, d_inner ? d_inner : T->inner_keys, ni, ext,
                                           T->nbr, T->parent, T->child, d_gflag, d_err);
  size_t tsc = 0;
  OCTMG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tsc, d_gflag, d_gscan, nl * 3, s));
  void* d_t3;
  OCTMG_TRY(dalloc(tmp, (char**)&d_t3, tsc));
  OCTMG_CUDA(cub::DeviceScan::ExclusiveSum(d_t3, tsc, d_gflag, d_gscan, nl * 3, s));
  k_glayer<<<nblk(nl * 3, 256), 256, 0, s>>>(d_gflag, d_gscan, nl * 3, T->glayer);
  int g_last[2];
  OCTMG_CUDA(cudaMemcpyAsync(&g_last[0], d_gscan + nl * 3 - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(&g_last[1], d_gflag + nl * 3 - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  OCTMG_CUDA(cudaGetLastError());
  if (h_err & ERR_NOT_GRADED) { set_error("leaf tiles are not 2:1 face graded"); return OCTMG_E_NOT_GRADED; }
  T->n_glayers = g_last[0] + g_last[1];
  return OCTMG_OK;
}

}  // namespace octmg
