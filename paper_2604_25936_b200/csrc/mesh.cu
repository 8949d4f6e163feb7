// mesh.cu -- marching cubes on the query grid, standalone or fused slab by slab with the query path
// (meshes are extracted from the SDF on a 512^3 grid with
// Marching Cubes; reading R24 for the triangulation rule, which the paper does not give).
//
// Configuration tables are derived at load time from the cube geometry (mc_build_tables), not stored:
// corner v = x + 2y + 4z is inside iff sdf < 0; each face is walked counter-clockwise as seen from
// outside; a crossing edge reached from an outside corner starts a segment that ends at the next
// crossing of the walk (diagonal inside corners of a face stay separated; face-local, so watertight);
// segments chain into loops; each loop, started at its smallest edge id, becomes a triangle fan.
//
// k_marching_cubes: blocks walk cube rows; one thread per grid vertex column of a row (4 loads, the x + 1
// corners from the next lane), tables in shared memory; surface cubes are queued per warp in shared memory
// and emitted, one triangle per lane, when more than 32 are waiting (scan of the queue's triangle counts + one
// atomicAdd per flush; output order is therefore not deterministic; the triangle set is).  Vertices are interpolated from the edge's lower
// corner so both cubes sharing an edge produce the same bits.  Bound: HBM (4 B of sdf per
// grid vertex + 36 B per triangle).
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#include "sand_internal.h"

namespace sand {

__constant__ uint8_t c_mc_ntri[256];
__constant__ uint8_t c_mc_tri[256][15];   // up to 5 triangles x 3 edge ids
__constant__ uint8_t c_mc_edge[12][2];    // (lower corner, upper corner)

static void mc_build_tables(uint8_t ntri[256], uint8_t tri[256][15], uint8_t edge[12][2]) {
  int ne = 0;
  for (int a = 0; a < 3; ++a)
    for (int v = 0; v < 8; ++v)
      if (!((v >> a) & 1)) {
        edge[ne][0] = (uint8_t)v;
        edge[ne][1] = (uint8_t)(v | (1 << a));
        ++ne;
      }
  int edge_id[8][8];
  for (int p = 0; p < 8; ++p)
    for (int q = 0; q < 8; ++q) edge_id[p][q] = -1;
  for (int e = 0; e < 12; ++e) edge_id[edge[e][0]][edge[e][1]] = edge_id[edge[e][1]][edge[e][0]] = e;
  // faces: normal axis a, side s; in-face axes u = a+1, w = a+2 (mod 3) with e_u x e_w = e_a, so the
  // cycle (0,0) (1,0) (1,1) (0,1) in (u, w) is counter-clockwise about +e_a; reversed for side 0
  int face[6][4];
  for (int a = 0, f = 0; a < 3; ++a) {
    const int u = (a + 1) % 3, w = (a + 2) % 3;
    const int cu[4] = {0, 1, 1, 0}, cw[4] = {0, 0, 1, 1};
    for (int s = 0; s < 2; ++s, ++f)
      for (int k = 0; k < 4; ++k) {
        const int kk = s ? k : 3 - k;
        face[f][k] = (s << a) | (cu[kk] << u) | (cw[kk] << w);
      }
  }
  for (int c = 0; c < 256; ++c) {
    int next[12];
    for (int e = 0; e < 12; ++e) next[e] = -1;
    for (int f = 0; f < 6; ++f) {
      int ce[4], cin[4], m = 0;
      for (int k = 0; k < 4; ++k) {
        const int p = face[f][k], q = face[f][(k + 1) & 3];
        const int ip = (c >> p) & 1, iq = (c >> q) & 1;
        if (ip != iq) {
          ce[m] = edge_id[p][q];
          cin[m] = iq;   // walked from outside into inside
          ++m;
        }
      }
      for (int k = 0; k < m; ++k)
        if (cin[k]) next[ce[k]] = ce[(k + 1) % m];
    }
    bool used[12] = {};
    int nt = 0;
    for (int e0 = 0; e0 < 12; ++e0) {
      if (next[e0] < 0 || used[e0]) continue;
      int loop[12], k = 0;
      for (int e = e0; !used[e]; e = next[e]) {
        used[e] = true;
        loop[k++] = e;
      }
      for (int m = 1; m + 1 < k; ++m) {
        tri[c][3 * nt] = (uint8_t)loop[0];
        tri[c][3 * nt + 1] = (uint8_t)loop[m];
        tri[c][3 * nt + 2] = (uint8_t)loop[m + 1];
        ++nt;
      }
    }
    ntri[c] = (uint8_t)nt;
  }
}

cudaError_t mc_upload_tables() {
  // constant memory is per device: upload once for each device this process uses
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && ((done >> dev) & 1)) return cudaSuccess;
  uint8_t ntri[256], tri[256][15] = {}, edge[12][2];
  mc_build_tables(ntri, tri, edge);
  e = cudaMemcpyToSymbol(c_mc_ntri, ntri, sizeof ntri);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mc_tri, tri, sizeof tri);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mc_edge, edge, sizeof edge);
  if (e == cudaSuccess && dev < 64) done |= 1ull << dev;
  return e;
}

// Grid axis x_i = fl32(2 i / (R - 1) - 1), computed in double (reading R8).
__global__ void k_grid_axis(int R, float* __restrict__ axis) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < R) axis[i] = (float)(2.0 * (double)i / (double)(R - 1) - 1.0);
}

// Points of grid planes [k0, k0 + np): index (i + R j) + R^2 (k - k0), x fastest.
__global__ void k_grid_points(const float* __restrict__ axis, int R, int k0, int np, float* __restrict__ pts) {
  const long long n = (long long)R * R * np;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q % R), j = (int)((q / R) % R), k = k0 + (int)(q / ((long long)R * R));
    pts[3 * q] = axis[i];
    pts[3 * q + 1] = axis[j];
    pts[3 * q + 2] = axis[k];
  }
}

// Cubes (i, j, k), 0 <= i, j < R - 1, kc0 <= k < kc1, over an sdf buffer holding planes from kp0 on.
// A block walks cube rows (j, k) (grid-stride, no per-element index division); a thread is grid vertex
// column i of the row: it loads the 4 values at x = i of the row's two y rows and two z planes and takes
// the x = i + 1 values from the next lane (the last lane of a warp loads them itself), ~4 loads a cube.
constexpr int MC_QC = 64;   // queue capacity per warp (cubes); flushed when a push of 32 might not fit
__global__ void __launch_bounds__(256) k_marching_cubes(const float* __restrict__ sdf, int R, int kc0, int kc1,
                                                        int kp0, const float* __restrict__ axis,
                                                        float* __restrict__ tris, long long cap,
                                                        unsigned long long* __restrict__ counter) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R1 = R - 1;
  // per warp: queue of surface cubes waiting for emission (8 corner values, i | j << 16, k | case << 24) and the
  // inclusive scan of their triangle counts, filled at flush time
  __shared__ float s_q[8][8][MC_QC];
  __shared__ unsigned s_m0[8][MC_QC], s_m1[8][MC_QC];
  __shared__ int s_off[8][MC_QC];
  const long long R2 = (long long)R * R;
  const long long nrows = (long long)R1 * (kc1 - kc0);
  __shared__ uint8_t s_tri[256][15];   // tables in shared memory: per-thread (divergent) indices
  __shared__ uint8_t s_ntri[256];
  __shared__ uint8_t s_edge[12][2];
  for (int t = threadIdx.x; t < 256 * 15; t += blockDim.x) s_tri[t / 15][t % 15] = c_mc_tri[t / 15][t % 15];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) s_ntri[t] = c_mc_ntri[t];
  if (threadIdx.x < 24) s_edge[threadIdx.x >> 1][threadIdx.x & 1] = c_mc_edge[threadIdx.x >> 1][threadIdx.x & 1];
  __syncthreads();
  // corner value v of the current cube without dynamic register indexing
  auto corner = [](const float (&lo)[4], const float (&hi)[4], int v) {
    const int u = ((v >> 1) & 1) | (((v >> 2) & 1) << 1);
    const float a = u == 0 ? lo[0] : u == 1 ? lo[1] : u == 2 ? lo[2] : lo[3];
    const float b = u == 0 ? hi[0] : u == 1 ? hi[1] : u == 2 ? hi[2] : hi[3];
    return (v & 1) ? b : a;
  };
  // segments of 256 cube columns of a row, block-strided; the next segment's loads are issued before the
  // current one is processed (its compute, counter atomic and emission hide their latency)
  const unsigned nseg = (unsigned)((R + 255) / 256);
  const unsigned nsg = (unsigned)nrows * nseg;
  // position (segment in row, j, k) of the next segment to load, stepped by gridDim.x segments with carries (a
  // division per segment cost a quarter of the kernel's instructions)
  const unsigned dseg = gridDim.x % nseg, drow = gridDim.x / nseg;
  const int dj = (int)(drow % (unsigned)R1), dk = (int)(drow / (unsigned)R1);
  int pseg = (int)(blockIdx.x % nseg), pj = (int)((blockIdx.x / nseg) % (unsigned)R1),
      pk = kc0 + (int)((blockIdx.x / nseg) / (unsigned)R1);
  auto load = [&](float (&v)[4], float (&x)[4], int& j, int& k, int& i) {
    j = pj;
    k = pk;
    i = pseg * 256 + (int)threadIdx.x;
    pseg += (int)dseg;
    const int cy = pseg >= (int)nseg;
    pseg -= cy ? (int)nseg : 0;
    pj += dj + cy;
    const int cz = pj >= R1;
    pj -= cz ? R1 : 0;
    pk += dk + cz;
    const float* rowp = sdf + (long long)(k - kp0) * R2 + (long long)j * R;
    const bool inr = i < R, ext = inr && i + 1 < R && lane == 31;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = inr ? __ldg(rowp + i + (u >> 1) * R2 + (u & 1) * R) : 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = ext ? __ldg(rowp + i + 1 + (u >> 1) * R2 + (u & 1) * R) : 0.f;
  };
  int qn = 0;   // queued cubes (warp-uniform)
  auto flush = [&]() {
    if (qn == 0) return;
    __syncwarp();
    // inclusive scan of the queued cubes' triangle counts (two entries per lane)
    const int e0 = 2 * lane, e1 = 2 * lane + 1;
    const int n0 = e0 < qn ? s_ntri[s_m1[warp][e0] >> 24] : 0;
    const int n1 = e1 < qn ? s_ntri[s_m1[warp][e1] >> 24] : 0;
    int off = n0 + n1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += y;
    }
    s_off[warp][e0] = off - n1;
    s_off[warp][e1] = off;
    const int T = __shfl_sync(0xffffffffu, off, 31);
    unsigned long long wbase = 0;
    if (lane == 31) wbase = atomicAdd(counter, (unsigned long long)T);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    __syncwarp();
    for (int idx = lane; idx < T; idx += 32) {
      if ((long long)wbase + idx >= cap) break;
      int L = 0;   // owner entry: the first L with inclusive count off[L] > idx
#pragma unroll
      for (int st = MC_QC / 2; st; st >>= 1)
        if (s_off[warp][L + st - 1] <= idx) L += st;
      const unsigned m0 = s_m0[warp][L], m1 = s_m1[warp][L];
      const int cL = (int)(m1 >> 24);
      const int t = idx - (s_off[warp][L] - s_ntri[cL]);
      const int iL = (int)(m0 & 0xFFFFu), jL = (int)(m0 >> 16), kL = (int)(m1 & 0xFFFFFFu);
      float plo[4], phi[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { plo[u] = s_q[warp][u][L]; phi[u] = s_q[warp][4 + u][L]; }
      float* out = tris + 9 * ((long long)wbase + idx);
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int e = s_tri[cL][3 * t + m];
        const int v0 = s_edge[e][0], v1 = s_edge[e][1];
        const float a0 = corner(plo, phi, v0), a1 = corner(plo, phi, v1);
        const float tt = a0 / (a0 - a1);
        const float p0x = axis[iL + (v0 & 1)], p0y = axis[jL + ((v0 >> 1) & 1)], p0z = axis[kL + (v0 >> 2)];
        const float p1x = axis[iL + (v1 & 1)], p1y = axis[jL + ((v1 >> 1) & 1)], p1z = axis[kL + (v1 >> 2)];
        out[3 * m] = p0x + tt * (p1x - p0x);
        out[3 * m + 1] = p0y + tt * (p1y - p0y);
        out[3 * m + 2] = p0z + tt * (p1z - p0z);
      }
    }
    __syncwarp();
    qn = 0;
  };
  float nv[4], nx[4];
  int nj = 0, nk = 0, ni = 0;
  if (blockIdx.x < nsg) load(nv, nx, nj, nk, ni);
  for (unsigned sg = blockIdx.x; sg < nsg; sg += gridDim.x) {
    {
      float lo[4], xx[4];   // x = i: (y, z) = (0,0) (1,0) (0,1) (1,1); lane 31 also x = i + 1
#pragma unroll
      for (int u = 0; u < 4; ++u) { lo[u] = nv[u]; xx[u] = nx[u]; }
      const int j = nj, k = nk, i = ni;
      if (sg + gridDim.x < nsg) load(nv, nx, nj, nk, ni);
      const bool inr = i < R;
      float hi[4];   // x = i + 1
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[u] = __shfl_down_sync(0xffffffffu, lo[u], 1);
      const bool cube = inr && i + 1 < R;
      if (lane == 31) {
#pragma unroll
        for (int u = 0; u < 4; ++u) hi[u] = xx[u];
      }
      int c = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = ((u & 1) << 1) | ((u >> 1) << 2);   // corner of (y, z) = (u & 1, u >> 1) at x = 0
        c |= (lo[u] < 0.f) << v;
        c |= (hi[u] < 0.f) << (v | 1);
      }
      const int nt = cube ? s_ntri[c] : 0;
      const unsigned act = __ballot_sync(0xffffffffu, nt != 0);
      if (!act) continue;   // most warps meet no surface
      // queue the surface cubes (emitting per 32-cube segment would run the long emission path with the ~9
      // triangles such a segment holds on average: ncu, 80 of the kernel's 137 M warp instructions)
      if (nt) {
        const int pos = qn + __popc(act & ((1u << lane) - 1u));
#pragma unroll
        for (int u = 0; u < 4; ++u) { s_q[warp][u][pos] = lo[u]; s_q[warp][4 + u][pos] = hi[u]; }
        s_m0[warp][pos] = (unsigned)i | ((unsigned)j << 16);
        s_m1[warp][pos] = (unsigned)k | ((unsigned)c << 24);
      }
      qn += __popc(act);
      if (qn > MC_QC - 32) flush();
    }
  }
  flush();
}

cudaError_t launch_grid_axis(int R, float* axis, cudaStream_t st) {
  k_grid_axis<<<(R + 255) / 256, 256, 0, st>>>(R, axis);
  return cudaGetLastError();
}

cudaError_t launch_grid_points(const float* axis, int R, int k0, int np, float* pts, int num_sms, cudaStream_t st) {
  k_grid_points<<<num_sms * 8, 256, 0, st>>>(axis, R, k0, np, pts);
  return cudaGetLastError();
}

cudaError_t launch_marching_cubes(const float* sdf, int R, int kc0, int kc1, int kp0, const float* axis, float* tris,
                                  long long cap, unsigned long long* counter, int num_sms, cudaStream_t st) {
  const long long nrows = (long long)(R - 1) * (kc1 - kc0);
  if (nrows <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>(nrows, (long long)num_sms * 8);
  k_marching_cubes<<<(unsigned)blocks, 256, 0, st>>>(sdf, R, kc0, kc1, kp0, axis, tris, cap, counter);
  return cudaGetLastError();
}

}  // namespace sand
