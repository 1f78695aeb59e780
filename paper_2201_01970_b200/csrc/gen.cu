// Device assembly of the synthetic black-oil Jacobians (src/problems.py:113-155).
//
// The reference scatters link terms with np.add.at and sorts a COO; on the
// structured 7-point grid every row's blocks are known in closed form, so one
// thread per cell writes its row directly (block columns ascending: -z, -y,
// -x, diagonal, +x, +y, +z).  Every value is the reference's expression with
// the reference's operand order and separately rounded IEEE operations
// (-fmad=false), including the np.add.at accumulation order of the diagonal:
// first the links whose lower end is the cell (x, y, z), then the links whose
// upper end is the cell, ordered by the lower cell (z, y, x).  The random
// fields (numpy Generator draws) and np.exp are evaluated on the host.
#include "device.cuh"
#include "engine.h"
#include "nvtx.h"

namespace cprb {

struct GenGrid {
  int64_t nx, ny, nz, n;
};

__device__ __forceinline__ void cell_xyz(const GenGrid& g, int64_t i, int64_t& ix, int64_t& iy,
                                         int64_t& iz) {
  ix = i % g.nx;
  iy = (i / g.nx) % g.ny;
  iz = i / (g.nx * g.ny);
}

__global__ void k_gen_count(const GenGrid g, int64_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  int64_t ix, iy, iz;
  cell_xyz(g, i, ix, iy, iz);
  cnt[i] = 1 + (ix > 0) + (iy > 0) + (iz > 0) + (ix + 1 < g.nx) + (iy + 1 < g.ny) + (iz + 1 < g.nz);
}

// aniso[axis] * 2.0 / (1.0 / perm[a] + 1.0 / perm[b])   (harmonic mean)
__device__ __forceinline__ double trans_of(int axis, double pa, double pb) {
  const double an = axis == 2 ? 0.2 : 1.0;
  return (an * 2.0) / (1.0 / pa + 1.0 / pb);
}

__global__ void k_gen_assemble(const GenGrid g, double drift, const double* __restrict__ perm,
                               const double* __restrict__ conv_scale,
                               const double* __restrict__ couple, const int64_t* __restrict__ ptr,
                               int64_t* __restrict__ cols, double* __restrict__ vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  int64_t ix, iy, iz;
  cell_xyz(g, i, ix, iy, iz);
  const int64_t step[3] = {1, g.nx, g.nx * g.ny};
  const bool has_m[3] = {ix > 0, iy > 0, iz > 0};
  const bool has_p[3] = {ix + 1 < g.nx, iy + 1 < g.ny, iz + 1 < g.nz};
  const double pi = perm[i];
  // link terms: lower links (a = i - step, b = i) and upper links (a = i, b = i + step)
  double tr_m[3], cv_m[3], tr_p[3];
  for (int ax = 0; ax < 3; ++ax) {
    tr_m[ax] = cv_m[ax] = tr_p[ax] = 0.0;
    if (has_m[ax]) {
      const int64_t a = i - step[ax];
      tr_m[ax] = trans_of(ax, perm[a], pi);
      cv_m[ax] = conv_scale[a] * tr_m[ax];
    }
    if (has_p[ax]) tr_p[ax] = trans_of(ax, pi, perm[i + step[ax]]);
  }
  int64_t p = ptr[i];
  auto put = [&](int64_t col, const double (&b)[9]) {
    cols[p] = col;
    double* v = vals + p * 9;
#pragma unroll
    for (int e = 0; e < 9; ++e) v[e] = b[e];
    ++p;
  };
  // lower neighbours in ascending column order: -z, -y, -x
  for (int ax = 2; ax >= 0; --ax) {
    if (!has_m[ax]) continue;
    const double cv = cv_m[ax];
    double b[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    b[0] = -tr_m[ax];
    b[4] = -cv;
    b[8] = -0.8 * cv;
    b[3] = (-drift * 0.5) * cv;
    b[6] = (-drift * 0.3) * cv;
    put(i - step[ax], b);
  }
  {  // diagonal: accumulation + outflow (np.add.at order), drift couplings
    double pd = 0.05 * pi;
    for (int ax = 0; ax < 3; ++ax)
      if (has_p[ax]) pd = pd + tr_p[ax];
    double wd = 1.0, od = 1.0;
    for (int ax = 2; ax >= 0; --ax)
      if (has_m[ax]) {
        pd = pd + tr_m[ax];
        wd = wd + cv_m[ax];
        od = od + 0.8 * cv_m[ax];
      }
    const double* c = couple + i * 6;
    double b[9];
    b[0] = pd;
    b[1] = drift * c[0];
    b[2] = drift * c[1];
    b[3] = drift * c[2];
    b[4] = wd;
    b[5] = (drift * 0.2) * c[3];
    b[6] = drift * c[4];
    b[7] = (drift * 0.2) * c[5];
    b[8] = od;
    put(i, b);
  }
  // upper neighbours: +x, +y, +z (pressure diffusion only)
  for (int ax = 0; ax < 3; ++ax) {
    if (!has_p[ax]) continue;
    double b[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    b[0] = -tr_p[ax];
    put(i + step[ax], b);
  }
}

}  // namespace cprb

using namespace cprb;

extern "C" int cprb_gen_row_counts(int64_t nx, int64_t ny, int64_t nz, int64_t* cnt, void* stream) {
  const GenGrid g{nx, ny, nz, nx * ny * nz};
  if (g.n <= 0) return CPRB_OK;
  k_gen_count<<<(int)((g.n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(g, cnt);
  return check_launch("gen row counts");
}

extern "C" int cprb_gen_assemble(int64_t nx, int64_t ny, int64_t nz, double drift,
                                 const double* perm, const double* conv_scale,
                                 const double* couple, const int64_t* row_ptr, int64_t* cols,
                                 double* vals, void* stream) {
  const GenGrid g{nx, ny, nz, nx * ny * nz};
  if (g.n <= 0) return CPRB_OK;
  NvtxRange nv("gen_assemble");
  k_gen_assemble<<<(int)((g.n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      g, drift, perm, conv_scale, couple, row_ptr, cols, vals);
  return check_launch("gen assemble");
}
