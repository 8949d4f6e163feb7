// sand_internal.h -- device-side structures shared by libsand's kernels and its host code.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <vector>

#include "../../include/sand.h"

namespace sand {

constexpr int kTileM = 128;           // rows (points) per T-MLP tile = tcgen05 M
constexpr int kLookupThreads = 256;   // K1 / K2b block size
constexpr int kLookupChunk = 4096;    // points per K1 / K2b block (16 per thread, 4 x float4 groups)
constexpr int kMaxBins = SAND_MAX_L + 2;  // depths 0..L plus one bin for non-finite points

// Written by the scan kernel (K2a), read by the T-MLP kernels and by sand_get_stats.
// Tiles are ordered deepest depth first; tile t belongs to depth d iff tile_begin[d] <= t < tile_end[d].
struct QueryMeta {
  long long count[kMaxBins];      // points per bin (bin L+1 = non-finite)
  long long start[kMaxBins];      // first perm[] row of depth d (d >= 1)
  long long tile_begin[kMaxBins];
  long long tile_end[kMaxBins];
  long long total_tiles;
  long long tile_rows;            // rows per tile (128: 1-CTA / SIMT kernels, 256: CTA-pair kernel)
};

struct LookupParams {
  int dense;              // 1: dense grid (voxel or baked octree), 0: octree descent
  int level;
  int L;
  int cap;                // LOD cap (1..L)
  const uint8_t* grid;    // dense: G^3 depth
  const float* grid_far;  // dense: G^3 cached sdf or nullptr
  const uint32_t* nodes;  // octree
  const uint8_t* leaf_depth;
  const float* leaf_far;
  const uint32_t* top;    // octree descent: node payload reached at level top_level per 2^top_level cell
  int top_level;          // (a dense 8 MB start table: the descent resumes below it), or nullptr / 0
};

// Host-side launchers (lookup.cu)
cudaError_t launch_lookup(const float* pts, long long n, const LookupParams& lp, uint8_t* out_depth,
                          float* out_sdf, uint32_t* hist, long long nblk, cudaStream_t st);
// even_bins: round every depth bin up to an even number of tiles (empty padding tiles), so consecutive tile pairs
// (2u, 2u + 1) always share a depth (the slot-team kernel runs them side by side in its two slots)
cudaError_t launch_scan(const uint32_t* hist, long long nblk, int L, int tile_rows, int even_bins, uint32_t* offs,
                        QueryMeta* meta, unsigned long long* scratch, cudaStream_t st);
long long scan_scratch_words(long long nblk);   // u64 words of scratch launch_scan needs
cudaError_t launch_scatter(const uint8_t* depth, long long n, int L, const uint32_t* offs, uint32_t* perm,
                           long long nblk, cudaStream_t st);
cudaError_t launch_bake_octree(const uint32_t* nodes, const uint8_t* leaf_depth, const float* leaf_far,
                               int level, uint8_t* grid, float* grid_far, int* err_flag, cudaStream_t st);
cudaError_t launch_bake_top(const uint32_t* nodes, int top_level, uint32_t* top, cudaStream_t st);

// T-MLP parameters as the kernels consume them (built by sand_load_weights).
struct MlpDev {
  int L, H, tail;
  float omega0;
  // FP32 SIMT path: raw hidden weights [L-1][H][H] (row-major W_i[j][k]) and biases
  const float* w_hidden;     // (L-1)*H*H
  // BF16 tcgen05 path: pre-swizzled SW128 K-major image [L-1][KC][H rows][128 B]
  const void* w_image;
  // same BF16 tiles regrouped for the CTA-pair kernel: [L-1][2 CTA halves][KC][H/2 rows][128 B], so a CTA's
  // half of a layer is one contiguous run (bulk copies of 2 K-chunks)
  const void* w_image_pair;
  // FP32 tables (both paths):
  //   w1: float4[H] = (w0*W1[j][0], w0*W1[j][1], w0*W1[j][2], w0*b1[j])
  //   bias: [L-1][H] = w0 * b_i (i >= 2);  a: [L][H] tail (a_i or a_i0);
  //   a1: [L-1][H] (MULT, i >= 2);  c: [L];  c1: [L-1] (MULT)   -- in this order
  const float* tables;
  long long off_w1, off_bias, off_a, off_c, off_a1, off_c1, tables_floats;
  // CTA-pair kernel tables.  tmlp_tc2.cu (w0 and every bias folded into the MMA operands):
  //   a: [L][H] tail vectors (a_i or a_i0);  a1: [L-1][H] (MULT)
  //   c   : [L] tail biases (MULT: c_i0);  c1: [L] (MULT: c_i1 at index i-1, i >= 2)
  //   csum: [L+1] LINEAR: sum_{i <= d} c_i;  MULT: c_1 (d >= 1)
  // tmlp_tc3.cu (wide kernel) additionally keeps w0 * b_i interleaved with a_i: [L][H/2][b pair, a pair].
  const float* pair_tables;
  const void* w1_image;      // layer-1 split-BF16 B operand, [2 halves][H/2 rows][16 bf16] (l1_off layout)
  long long pt_floats, pt_off_l1, pt_off_bias, pt_off_a, pt_off_a1, pt_off_c, pt_off_c1, pt_off_csum;
  int kprof;                 // diagnostic (SAND_OPT_KPROF): per-role clock counters, synchronous dump
  // split-FP16 x3 kernel (tmlp_x3.cu, FP32-accurate on tensor cores): per (layer, CTA) image
  // [split bias][KC W_hi chunks][KC W_lo chunks] and FP32 tables: w1 float4 [H] (w0 W1, w0 b1), a [L][H],
  // a1 [L-1][H] (MULT), c [L], c1 [L]
  const void* x3_image;
  const float* x3_tables;
  // slot-team CTA-pair kernel (tmlp_tc4.cu): layer-1 split-BF16 operand [2 CTAs][H/2 rows][16 bf16] and
  // per (layer, CTA) runs [bias operand][KC SW128 K-chunks] of this CTA's H/2 output features; tables = pair_tables
  const void* tc4_w1;
  const void* tc4_image;
  long long x3_floats, x3_off_w1, x3_off_a, x3_off_a1, x3_off_c, x3_off_c1;
};


cudaError_t launch_tmlp_simt(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                             float* out_sdf, int num_sms, cudaStream_t st);
// pair_mode (SAND_OPT_PAIR_KERNEL): 0 = 1-CTA kernel; 1 = two-pass CTA-pair kernel (tc2 / tc3);
// 2 = slot-team CTA-pair kernel (tc4) where usable, else as 1.  Pair kernels consume 256-row tiles.
cudaError_t launch_tmlp_tc(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                           float* out_sdf, int num_sms, cudaStream_t st, int pair_mode);
// configuration query: dynamic smem bytes for the tc kernel, 0 if unsupported
size_t tc_smem_bytes(int L, int H, int tail);
int tmlp_tile_rows(int H, int prec, int pair_mode);   // tile size the selected T-MLP kernel consumes
bool tc_supported_H(int H);
bool simt_supported_H(int H);
size_t simt_smem_bytes(int L, int H, int tail);
cudaError_t prepare_tmlp_kernels(int L, int H, int tail, int prec);
// depth-map population (depthpop.cu)
bool depthpop_supported(int H);
// Marching cubes (mesh.cu)
cudaError_t mc_upload_tables();
cudaError_t launch_grid_axis(int R, float* axis, cudaStream_t st);
cudaError_t launch_grid_points(const float* axis, int R, int k0, int np, float* pts, int num_sms, cudaStream_t st);
size_t mc_counter_words();                 // uint64 words of the counter block (triangle count + pass B's task counters)
size_t mc_sign_words(int R, int planes);   // scratch (uint32 words) for the vertex signs of `planes` grid planes
cudaError_t launch_marching_cubes(const float* sdf, int R, int kc0, int kc1, int kp0, const float* axis, float* tris,
                                  long long cap, unsigned long long* counter, uint32_t* signs, int num_sms,
                                  cudaStream_t st);
// hbuf: per-block activation scratch (dynamic_scratch_floats) -> pool kernel with re-compaction;
// nullptr -> tile-level early exit
cudaError_t launch_query_dynamic(const MlpDev& m, const float* w_t, const float* pts, long long n, float r,
                                 float* out_sdf, uint8_t* out_depth, float* hbuf, int num_sms, cudaStream_t st);
size_t dynamic_scratch_floats(int H, int num_sms);
// FP32 adaptive query for H in {128, 256, 336} (binned 128-row tiles; depthpop.cu)
bool query_fp32_supported(int H);
cudaError_t launch_query_fp32(const MlpDev& m, const float* w_t, const float* pts, const uint32_t* perm,
                              const QueryMeta* meta, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_required_depth(const MlpDev& m, const float* w_t, const float* pts, long long n, float r,
                                  int near, uint8_t* out, int num_sms, cudaStream_t st);
cudaError_t launch_leaf_max(const uint8_t* d, long long n_leaves, int spl, uint8_t* out, cudaStream_t st);
// CTA-pair kernel (tmlp_tc2.cu)
bool tc2_available(int H);
bool tc2_usable(int L, int H, int tail);           // H supported and the kernel's shared memory fits
void tc2_table_layout(int L, int H, int tail, MlpDev* m, bool interleave);   // pair-table offsets (pt_off_*, pt_floats)
// host images of the CTA-pair kernel: tables, layer-1 split-BF16 operand, per-(layer, half) bias + weight image
void tc2_build_host(int L, int H, int tail, float w0, const float* const* W, const float* const* b,
                    const float* const* a, const float* const* a1, const float* c, const float* c1, MlpDev* m,
                    std::vector<float>* tables, std::vector<uint16_t>* w1img, std::vector<uint8_t>* img);
cudaError_t launch_tmlp_tc2(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st);
cudaError_t prepare_tc2(int H, int tail);
// Slot-team CTA-pair kernel (tmlp_tc4.cu): one N = H MMA chain per layer, one epilogue team per tile slot
bool tc4_available(int H, int tail);
bool tc4_usable(int L, int H, int tail);
bool tc4_runs(int L, int H, int tail, int prec, int pair_mode);   // launch_tmlp_tc would pick the slot-team kernel
void tc4_build_host(int L, int H, float w0, const float* const* W, const float* const* b, std::vector<uint16_t>* w1img,
                    std::vector<uint8_t>* img);
cudaError_t launch_tmlp_tc4(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st);
cudaError_t prepare_tc4(int H, int tail);
size_t tc2_w1_offset(int H, int n, int k);   // byte offset of (unit n, column k) in MlpDev::w1_image
// Wide CTA-pair kernel (tmlp_tc3.cu): H = 336, LINEAR; one 256-row tile split into two N-halves.  It reuses
// MlpDev::pair_tables / w1_image / w_image_pair with its own (padded-width) layouts, built by tc3_build_host.
bool tc3_available(int H, int tail);
bool tc3_usable(int L, int H, int tail);
void tc3_build_host(int L, int H, float w0, const float* const* W, const float* const* b, const float* const* a,
                    const float* c, MlpDev* m, std::vector<float>* tables, std::vector<uint16_t>* w1img,
                    std::vector<uint8_t>* img);
cudaError_t launch_tmlp_tc3(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta,
                            float* out, int num_sms, cudaStream_t st);
cudaError_t prepare_tc3();
// FP32-accurate CTA-pair kernel on split-FP16 operands (tmlp_x3.cu): query and Eq. 5 population modes
bool x3_available(int H);
bool x3_usable(int L, int H, int tail, int pop);
void x3_build_host(int L, int H, int tail, float w0, const float* const* W, const float* const* b,
                   const float* const* a, const float* const* a1, const float* c, const float* c1, MlpDev* m,
                   std::vector<float>* tables, std::vector<uint8_t>* img);
cudaError_t launch_tmlp_x3(const MlpDev& m, const float* pts, const uint32_t* perm, const QueryMeta* meta, float* out,
                           int num_sms, cudaStream_t st);
cudaError_t launch_required_depth_x3(const MlpDev& m, const float* pts, long long n, float r, int near, uint8_t* out,
                                     int num_sms, cudaStream_t st);
cudaError_t launch_query_dynamic_x3(const MlpDev& m, const float* pts, long long n, float r, float* out_sdf,
                                    uint8_t* out_depth, int num_sms, cudaStream_t st);

}  // namespace sand
