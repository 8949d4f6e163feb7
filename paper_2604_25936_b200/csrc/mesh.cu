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
// Two kernels (below): k_mc_signs packs the vertex signs into words, k_mc_emit finds the surface cubes with
// word-wide bit operations, queues them per warp in shared memory and emits a full queue's triangles one per
// lane (scan of the queue's triangle counts + one atomicAdd per flush; output order is therefore not
// deterministic; the triangle set is).  Vertices are interpolated from the edge's lower
// corner so both cubes sharing an edge produce the same bits.  Bound: HBM (4 B of sdf per
// grid vertex + 36 B per triangle).
#include <algorithm>
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

#include "sand_internal.h"

namespace sand {

// device-global (not __constant__): every block copies them to shared memory with coalesced word loads
__device__ __align__(16) uint8_t c_mc_ntri[256];
__device__ __align__(16) uint16_t c_mc_tri[256][5];   // up to 5 triangles: edge ids e0 | e1 << 4 | e2 << 8
__device__ __align__(16) uint8_t c_mc_edge[16];       // per edge: lower corner | axis << 3 (upper corner = lower | 1 << axis)

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
  uint16_t tri16[256][5] = {};
  for (int c = 0; c < 256; ++c)
    for (int t = 0; t < ntri[c]; ++t)
      tri16[c][t] = (uint16_t)(tri[c][3 * t] | (tri[c][3 * t + 1] << 4) | (tri[c][3 * t + 2] << 8));
  uint8_t edge8[16] = {};
  for (int k = 0; k < 12; ++k) {
    int a = 0;
    while ((edge[k][0] | (1 << a)) != edge[k][1]) ++a;   // mc_build_tables: upper = lower | 1 << axis
    edge8[k] = (uint8_t)(edge[k][0] | (a << 3));
  }
  e = cudaMemcpyToSymbol(c_mc_ntri, ntri, sizeof ntri);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mc_tri, tri16, sizeof tri16);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mc_edge, edge8, sizeof edge8);
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

// ---- marching cubes in two passes over an sdf buffer holding planes from kp0 on.
//
// Pass A (k_mc_signs): the sign of every grid vertex as a bit.  Row = (plane, y) line of R vertices; per group
// of 128 vertices four words m_0..m_3, bit L of m_q = sdf(vertex 128 g + 4 L + q) < 0 -- the layout a lane
// that loads 4 consecutive vertices (16 bytes) produces with four ballots.  HBM-bound: 4 B read per vertex.
//
// Pass B (k_mc_emit): a thread takes (group g, cube row j, plane k) = 128 cubes, finds the cubes that meet
// the surface with word-wide bit operations on 4 rows' words (x + 1 is the next q, or the next lane bit for
// q = 3), and queues them per warp in shared memory; a full queue is flushed: corner values gathered from
// the sdf (2 queue entries per lane), scan of the triangle counts, one atomicAdd, triangles emitted one per
// lane.  Only ~2.5% of the cubes of the 512^3 grid meet the surface, so pass B touches the sdf only there.
#ifndef SAND_MC_UNROLL
#define SAND_MC_UNROLL 2   // emission iterations interleaved (the loop body is one long dependent chain)
#endif
#ifndef SAND_MC_QC
#define SAND_MC_QC 64    // 128 measured 6-9% slower (47 KB of shared memory per block, 7-step owner search)
#endif
constexpr int MC_UNROLL = SAND_MC_UNROLL;
// Pass B's work queue: MC_NRANGE task ranges, each with its own counter on its own 128-byte line (a single
// counter next to the triangle counter serialised ~200 K same-sector atomics: 340 us of pass B on the 512^3 grid)
constexpr int MC_NRANGE = 64;
constexpr int MC_CTR_STRIDE = 16;   // uint64 words between counters
constexpr int MC_QC = SAND_MC_QC;   // queue capacity per warp (cubes), a multiple of 32
constexpr int MC_EPL = MC_QC / 32;  // queue entries per lane at flush time

__global__ void __launch_bounds__(256) k_mc_signs(const float* __restrict__ sdf, int R, long long nrows, int G,
                                                  uint32_t* __restrict__ signs, unsigned long long* __restrict__ taskctr) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < MC_NRANGE) taskctr[MC_CTR_STRIDE * threadIdx.x] = 0ull;   // pass B's work queue (same stream, runs after this)
  const bool al = (R & 3) == 0 && (reinterpret_cast<uintptr_t>(sdf) & 15) == 0;
  const long long ngr = nrows * G;
  const long long wstride = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long gi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < ngr; gi += wstride) {
    const long long row = gi / G;
    const int x = (int)(gi - row * G) * 128 + 4 * lane;
    const float* rp = sdf + row * R + x;
    float v[4];
    if (al && x < R) {
      const float4 t = __ldcs(reinterpret_cast<const float4*>(rp));
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = x + q < R ? __ldcs(rp + q) : 0.f;
    }
    uint32_t m[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) m[q] = __ballot_sync(0xffffffffu, v[q] < 0.f);
    if (lane == 0) *reinterpret_cast<uint4*>(signs + 4 * gi) = make_uint4(m[0], m[1], m[2], m[3]);
  }
}

__global__ void __launch_bounds__(256, 4) k_mc_emit(const float* __restrict__ sdf, const uint32_t* __restrict__ signs,
                                                    int R, int kc0, int kc1, int kp0, const float* __restrict__ axis,
                                                    float* __restrict__ tris, long long cap,
                                                    unsigned long long* __restrict__ counter,
                                                    unsigned long long* __restrict__ taskctr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int R1 = R - 1;
  const int G = (R + 127) / 128;
  const long long R2 = (long long)R * R;
  // per warp: queue of surface cubes waiting for emission (x | j << 16, k | case << 24), their 8 corner values
  // and the inclusive scan of their triangle counts, both filled at flush time
  __shared__ float s_q[8][8][MC_QC];
  __shared__ unsigned s_m0[8][MC_QC], s_m1[8][MC_QC];
  __shared__ unsigned short s_off[8][MC_QC];   // <= 5 MC_QC triangles
  __shared__ __align__(16) uint16_t s_tri[256][5];   // tables in shared memory: per-thread (divergent) indices
  __shared__ __align__(16) uint8_t s_ntri[256];
  __shared__ __align__(16) uint8_t s_edge[16];
  for (int t = threadIdx.x; t < 256 * 5 / 2; t += blockDim.x)
    reinterpret_cast<uint32_t*>(&s_tri[0][0])[t] = reinterpret_cast<const uint32_t*>(&c_mc_tri[0][0])[t];
  if (threadIdx.x < 64) reinterpret_cast<uint32_t*>(s_ntri)[threadIdx.x] = reinterpret_cast<const uint32_t*>(c_mc_ntri)[threadIdx.x];
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(s_edge)[threadIdx.x] = reinterpret_cast<const uint32_t*>(c_mc_edge)[threadIdx.x];
  __syncthreads();
  int qn = 0;   // queued cubes (warp-uniform)
  auto flush = [&]() {
    if (qn == 0) return;
    __syncwarp();
    int nh[MC_EPL];   // triangle counts of this lane's entries MC_EPL lane + h
    int off = 0;
#pragma unroll
    for (int h = 0; h < MC_EPL; ++h) {
      nh[h] = MC_EPL * lane + h < qn ? s_ntri[s_m1[warp][MC_EPL * lane + h] >> 24] : 0;
      off += nh[h];
    }
    const int mine = off;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += y;
    }
    {
      int run = off - mine;   // inclusive scan over the queue entries
#pragma unroll
      for (int h = 0; h < MC_EPL; ++h) {
        run += nh[h];
        s_off[warp][MC_EPL * lane + h] = (unsigned short)run;
      }
    }
    const int T = __shfl_sync(0xffffffffu, off, 31);
    unsigned long long wbase = 0;
    if (lane == 31) wbase = atomicAdd(counter, (unsigned long long)T);   // in flight under the corner gather
#pragma unroll
    for (int h = 0; h < MC_EPL; ++h) {   // gather the corners of this lane's entries
      const int e = MC_EPL * lane + h;
      if (e < qn) {
        const unsigned m0 = s_m0[warp][e], m1 = s_m1[warp][e];
        const float* cp = sdf + (long long)((int)(m1 & 0xFFFFFFu) - kp0) * R2 + (long long)(m0 >> 16) * R + (m0 & 0xFFFFu);
#pragma unroll
        for (int u = 0; u < 4; ++u) {   // (y, z) = (u & 1, u >> 1)
          const float* q = cp + (u >> 1) * R2 + (u & 1) * R;
          s_q[warp][u][e] = __ldg(q);
          s_q[warp][4 + u][e] = __ldg(q + 1);
        }
      }
    }
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    __syncwarp();
#pragma unroll MC_UNROLL
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
      float* out = tris + 9 * ((long long)wbase + idx);
      const unsigned pk = s_tri[cL][t];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        // vertex on edge e: from its lower corner v0 along axis ax; t = s0 / (s0 - s1) (R24).  The other two
        // coordinates are the lower corner's own (p0 + t * 0), so only the edge axis is interpolated.
        const unsigned eb = s_edge[(pk >> (4 * m)) & 15u];
        const int v0 = (int)(eb & 7u), ax = (int)(eb >> 3), v1 = v0 | (1 << ax);
        // corner v = x + 2 y + 4 z is queue row 4 x + (v >> 1)
        const float a0 = s_q[warp][4 * (v0 & 1) + (v0 >> 1)][L], a1 = s_q[warp][4 * (v1 & 1) + (v1 >> 1)][L];
        const float tt = __fdividef(a0, a0 - a1);
        const int i0 = iL + (v0 & 1), j0 = jL + ((v0 >> 1) & 1), k0 = kL + (v0 >> 2);
        float px = axis[i0], py = axis[j0], pz = axis[k0];
        const float pe0 = ax == 0 ? px : ax == 1 ? py : pz;
        const float pe1 = axis[(ax == 0 ? i0 : ax == 1 ? j0 : k0) + 1];
        const float pe = pe0 + tt * (pe1 - pe0);
        if (ax == 0) px = pe;
        else if (ax == 1) py = pe;
        else pz = pe;
        out[3 * m] = px;
        out[3 * m + 1] = py;
        out[3 * m + 2] = pz;
      }
    }
    __syncwarp();
    qn = 0;
  };
  // lane task = one sign word: 32 cubes x = 128 g + 4 L + q (L = bit) of cube row j, plane k; warp tasks of 32
  // lane tasks are handed out by a global counter (surface-dense tasks run up to 16 flushes, empty ones none)
  const long long ntask = 4ll * G * R1 * (kc1 - kc0);
  const long long nwt = (ntask + 31) >> 5;
  // range r holds the warp tasks t = r (mod MC_NRANGE), so all ranges carry the same mix of dense and empty tasks
  // and run dry together; lane 0 draws tickets from its warp's home range and, once that is dry, from the next
  // two (a longer walk would only add dependent atomics to the kernel's tail)
  int rg = (int)(((long long)blockIdx.x * 8 + warp) % MC_NRANGE), dry = 0;
  auto issue = [&]() { return (long long)atomicAdd(taskctr + MC_CTR_STRIDE * rg, 1ull); };
  auto resolve = [&](long long raw) {   // ticket of range rg -> warp task, or -1 when the warp is done
    while (true) {
      const long long t = raw * MC_NRANGE + rg;
      if (t < nwt) return t;
      if (++dry >= 3) return -1ll;
      rg = rg + 1 == MC_NRANGE ? 0 : rg + 1;
      raw = issue();
    }
  };
  long long wt = 0;
  if (lane == 0) wt = resolve(issue());
  wt = __shfl_sync(0xffffffffu, wt, 0);
  while (wt >= 0) {
    long long nxt = 0;
    if (lane == 0) nxt = issue();   // next ticket, fetched under this task
    const long long t = wt * 32 + lane;
    const bool valid = t < ntask;
    const int q = (int)(t & 3);
    const long long tg = valid ? t >> 2 : 0;
    const int g = (int)(tg % G);
    const long long rest = tg / G;
    const int j = (int)(rest % R1), k = kc0 + (int)(rest / R1);
    uint32_t a[4] = {}, b[4] = {};   // [row u = (y, z)]: vertices x (a) and x + 1 (b) as bit L
    if (valid) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const long long row = (long long)(k - kp0 + (u >> 1)) * R + (j + (u & 1));
        const uint32_t* w = signs + 4 * (row * G + g);
        a[u] = __ldg(w + q);
        if (q < 3) b[u] = __ldg(w + q + 1);
        else b[u] = (__ldg(w) >> 1) | ((g + 1 < G ? __ldg(w + 4) : 0u) << 31);
      }
    }
    uint32_t m = 0;   // cubes with a sign change among their 8 corners
#pragma unroll
    for (int u = 0; u < 4; ++u) m |= (a[u] ^ a[0]) | (b[u] ^ a[0]);
    // cubes need x + 1 <= R - 1: x = 128 g + 4 L + q < R1  <=>  L < (R1 - 128 g - q + 3) / 4
    const int nl = (R1 - 128 * g - q + 3) >> 2;
    m &= nl >= 32 ? 0xFFFFFFFFu : (nl <= 0 ? 0u : ((1u << nl) - 1u));
    if (!valid) m = 0;
    while (__any_sync(0xffffffffu, m != 0)) {
      const int cnt = __popc(m);
      int off = cnt;   // inclusive scan of the lanes' pending cubes
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += y;
      }
      // lanes whose cubes still fit form a prefix (off is monotone)
      const bool fits = off <= MC_QC - qn;
      const unsigned fm = __ballot_sync(0xffffffffu, fits);
      const int nfit = __popc(fm);
      const int pushed = nfit ? __shfl_sync(0xffffffffu, off, nfit - 1) : 0;
      if (fits && m) {
        int pos = qn + off - cnt;
        while (m) {
          const int L = __ffs(m) - 1;
          m &= m - 1;
          unsigned c = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int v = ((u & 1) << 1) | ((u >> 1) << 2);   // corner (0, y, z)
            c |= ((a[u] >> L) & 1u) << v;
            c |= ((b[u] >> L) & 1u) << (v | 1);
          }
          s_m0[warp][pos] = (unsigned)(128 * g + 4 * L + q) | ((unsigned)j << 16);
          s_m1[warp][pos] = (unsigned)k | (c << 24);
          ++pos;
        }
      }
      qn += pushed;
      if (__any_sync(0xffffffffu, m != 0)) flush();   // something did not fit
    }
    if (lane == 0) nxt = resolve(nxt);
    wt = __shfl_sync(0xffffffffu, nxt, 0);
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

size_t mc_counter_words() { return (size_t)MC_CTR_STRIDE * (1 + MC_NRANGE); }   // uint64: triangle count + task counters
size_t mc_sign_words(int R, int planes) { return (size_t)4 * ((R + 127) / 128) * (size_t)R * (size_t)planes; }

// signs: scratch of mc_sign_words(R, kc1 - kc0 + 1) uint32 (16-byte aligned)
cudaError_t launch_marching_cubes(const float* sdf, int R, int kc0, int kc1, int kp0, const float* axis, float* tris,
                                  long long cap, unsigned long long* counter, uint32_t* signs, int num_sms,
                                  cudaStream_t st) {   // counter: mc_counter_words() uint64 (triangle count, task counters)
  if (R < 2 || kc1 <= kc0) return cudaSuccess;
  if (R > 65535) return cudaErrorInvalidValue;   // queue entries pack x and j into 16 bits each
  const int G = (R + 127) / 128;
  // planes kc0 .. kc1 of the buffer (it starts at plane kp0); their sign words are indexed from plane kp0 too
  const long long row0 = (long long)(kc0 - kp0) * R, nrows = (long long)(kc1 - kc0 + 1) * R;
  const long long ngr = nrows * G;
  const long long ba = std::min<long long>((ngr + 7) / 8, (long long)num_sms * 16);
  k_mc_signs<<<(unsigned)ba, 256, 0, st>>>(sdf + row0 * R, R, nrows, G, signs + 4 * row0 * G, counter + MC_CTR_STRIDE);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long long nwt = (4ll * G * (R - 1) * (kc1 - kc0) + 31) / 32;
  const long long bb = std::min<long long>((nwt + 7) / 8, (long long)num_sms * 4);
  k_mc_emit<<<(unsigned)bb, 256, 0, st>>>(sdf, signs, R, kc0, kc1, kp0, axis, tris, cap, counter, counter + MC_CTR_STRIDE);
  return cudaGetLastError();
}

}  // namespace sand
