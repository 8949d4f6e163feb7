// sand_api.cu -- host implementation of the libsand C ABI (include/sand.h).
//
// Owns the per-context device state: converted T-MLP parameters (FP32 tables, BF16 tcgen05 weight
// image), the depth map (dense grid or octree), the query workspace (histograms, scan offsets, the
// perm[] binning array, QueryMeta) and CUDA events for the per-stage timings.  Every compute step of
// a query runs in libsand's own kernels (lookup.cu, tmlp_tc.cu, tmlp_simt.cu); there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/sand.h"
#include "sand_internal.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for nsys / ncu timelines, inert without a tool

using namespace sand;

// Host-side NVTX range (enqueue of a library stage) -- SURVEY 5's profiling aux.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct sand_ctx {
  sand_config cfg{};
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  int lod_cap = 0;
  int use_pair = 2;       // SAND_OPT_PAIR_KERNEL: 0 = 1-CTA, 1 = two-pass CTA-pair, 2 = slot-team CTA-pair kernel
  bool pair_ok = true;    // a CTA-pair kernel supports (L, H, tail) at all
  bool team_ok = false;   // the slot-team CTA-pair kernel does
  int dyn_schedule = 0;   // sand_query_dynamic schedule (SAND_OPT_DYN_SCHEDULE)
  int kprof = 0;          // diagnostic per-role counters (SAND_OPT_KPROF)
  std::string err;
  // weights
  bool have_w = false;
  float* d_tables = nullptr;
  float* d_pair_tables = nullptr;
  void* d_w1_image = nullptr;
  void* d_wimage = nullptr;
  void* d_wimage_pair = nullptr;
  void* d_tc4_w1 = nullptr;       // slot-team kernel images (tmlp_tc4.cu)
  void* d_tc4_image = nullptr;
  float* d_whidden = nullptr;
  float* d_wt_f32 = nullptr;      // FP32 hidden weights transposed [L-1][k][j] (depth-map population)
  void* d_x3_image = nullptr;     // split-FP16 hidden-layer image (tmlp_x3.cu)
  float* d_x3_tables = nullptr;
  bool have_x3 = false;
  int fp32_tensor = 1;            // SAND_OPT_FP32_TENSOR
  uint8_t* d_dp_tmp = nullptr;    // per-sample depths of sand_populate_leaf_depths
  long long cap_dp = 0;
  // marching cubes (mesh.cu): grid axis, slab buffers of the fused extraction, triangle counter
  float* d_axis = nullptr;
  int axis_R = 0;
  float* d_mpts = nullptr;
  float* d_msdf = nullptr;
  uint8_t* d_mdep = nullptr;
  long long cap_m = 0;
  unsigned long long* d_tricount = nullptr;
  uint32_t* d_msigns = nullptr;   // vertex sign words of the planes one marching-cubes launch covers
  size_t cap_msigns = 0;
  float* d_dyn_h = nullptr;       // dynamic-exit activation scratch (per block, kDynPool x HP floats)
  MlpDev mlp{};
  // depth map
  bool have_dm = false;
  LookupParams lp{};
  uint8_t* d_grid = nullptr;
  float* d_grid_far = nullptr;
  uint32_t* d_top = nullptr;   // octree start table (levels > 8)
  uint32_t* d_nodes = nullptr;
  uint8_t* d_leaf_depth = nullptr;
  float* d_leaf_far = nullptr;
  // workspace
  long long cap_n = 0, cap_nblk = 0;
  uint32_t* d_hist = nullptr;
  uint32_t* d_offs = nullptr;
  unsigned long long* d_scan = nullptr;
  uint32_t* d_perm = nullptr;
  QueryMeta* d_meta = nullptr;
  // timing: one event quad per query since the last sand_get_stats (grown on demand; never
  // synchronised inside sand_query, so back-to-back queries stay asynchronous)
  std::vector<std::array<cudaEvent_t, 4>> evq;
  size_t nq = 0;      // quads used since the last sand_get_stats
  size_t last_q = 0;  // quad of the last query
  bool have_stats = false;
  long long last_n = 0;
  // host-buffer pipeline
  long long cap_h = 0;
  float* d_hpts[2] = {nullptr, nullptr};
  float* d_hsdf[2] = {nullptr, nullptr};
  uint8_t* d_hdep[2] = {nullptr, nullptr};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr, s_cmp = nullptr;
  cudaEvent_t e_in[2] = {nullptr, nullptr}, e_done[2] = {nullptr, nullptr}, e_out[2] = {nullptr, nullptr};
};

static thread_local std::string g_create_err;

static int fail(sand_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_create_err = buf;
  return code;
}

#define CU(call)                                                                                       \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? SAND_ERR_OOM : SAND_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                                  \
  } while (0)

template <class T>
static void dfree(T*& p) {
  if (p) cudaFree((void*)p);
  p = nullptr;
}

static bool supported(const sand_config& c) {
  if (c.prec == SAND_FP32)
    return (simt_supported_H(c.H) && simt_smem_bytes(c.L, c.H, c.tail) <= 232448) ||
           (query_fp32_supported(c.H) && c.L <= 32);
  if (c.prec == SAND_BF16)
    return tc_supported_H(c.H) && (tc2_usable(c.L, c.H, c.tail) || tc3_usable(c.L, c.H, c.tail) ||
                                   tc_smem_bytes(c.L, c.H, c.tail) > 0);
  if (c.prec == SAND_F16X3) return x3_usable(c.L, c.H, c.tail, 0);
  return false;
}

extern "C" int sand_abi_version(void) { return SAND_ABI_VERSION; }

extern "C" const char* sand_last_error(const sand_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

extern "C" int sand_create(const sand_config* cfg, sand_ctx** out) {
  sand_ctx* ctx = nullptr;
  if (!cfg || !out) return fail(nullptr, SAND_ERR_ARG, "sand_create: NULL argument");
  if (cfg->L < 1 || cfg->L > SAND_MAX_L) return fail(nullptr, SAND_ERR_ARG, "L=%d outside [1,%d]", cfg->L, SAND_MAX_L);
  if (!(cfg->omega0 > 0.0f) || !std::isfinite(cfg->omega0)) return fail(nullptr, SAND_ERR_ARG, "omega0 must be > 0");
  if (cfg->H < 1) return fail(nullptr, SAND_ERR_ARG, "H must be positive");
  if (cfg->tail != SAND_TAIL_LINEAR && cfg->tail != SAND_TAIL_MULT) return fail(nullptr, SAND_ERR_ARG, "bad tail mode");
  if (cfg->prec != SAND_FP32 && cfg->prec != SAND_BF16 && cfg->prec != SAND_TF32X3 && cfg->prec != SAND_F16X3)
    return fail(nullptr, SAND_ERR_ARG, "bad precision");
  if (!supported(*cfg))
    return fail(nullptr, SAND_ERR_UNSUPPORTED, "unsupported (precision %d, L %d, H %d, tail %d)", (int)cfg->prec,
                cfg->L, cfg->H, (int)cfg->tail);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(nullptr, SAND_ERR_CUDA, "no CUDA device available (libsand has no CPU path)");
  if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, SAND_ERR_ARG, "device %d out of range", cfg->device);
  ctx = new (std::nothrow) sand_ctx();
  if (!ctx) return fail(nullptr, SAND_ERR_OOM, "host allocation failed");
  ctx->cfg = *cfg;
  ctx->lod_cap = cfg->L;
  auto bail = [&](int code) { g_create_err = ctx->err; sand_destroy(ctx); return code; };
  if (cudaSetDevice(cfg->device) != cudaSuccess) { fail(ctx, SAND_ERR_CUDA, "cudaSetDevice failed"); return bail(SAND_ERR_CUDA); }
  cudaDeviceProp prop{};
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess) { fail(ctx, SAND_ERR_CUDA, "cudaGetDeviceProperties failed"); return bail(SAND_ERR_CUDA); }
  if (prop.major != 10) {
    fail(ctx, SAND_ERR_UNSUPPORTED, "libsand is built for sm_100a (B200); device is sm_%d%d", prop.major, prop.minor);
    return bail(SAND_ERR_UNSUPPORTED);
  }
  ctx->num_sms = prop.multiProcessorCount;
  // the CTA-pair kernel keeps its per-column tables in shared memory: large L falls back to the 1-CTA kernel
  if (cfg->prec == SAND_BF16)
  {
    ctx->pair_ok = tc2_usable(cfg->L, cfg->H, cfg->tail) || tc3_usable(cfg->L, cfg->H, cfg->tail);
    ctx->team_ok = tc4_usable(cfg->L, cfg->H, cfg->tail);
  }
  ctx->use_pair = ctx->team_ok ? 2 : (ctx->pair_ok ? 1 : 0);
  cudaError_t e = prepare_tmlp_kernels(cfg->L, cfg->H, cfg->tail, cfg->prec);
  if (e != cudaSuccess) { fail(ctx, SAND_ERR_CUDA, "kernel attribute setup: %s", cudaGetErrorString(e)); return bail(SAND_ERR_CUDA); }
  *out = ctx;
  return SAND_OK;
}

static void free_workspace(sand_ctx* c) {
  dfree(c->d_hist); dfree(c->d_offs); dfree(c->d_scan); dfree(c->d_perm); dfree(c->d_meta);
  c->cap_n = c->cap_nblk = 0;
}
static void free_depthmap(sand_ctx* c) {
  dfree(c->d_grid); dfree(c->d_grid_far); dfree(c->d_top); dfree(c->d_nodes); dfree(c->d_leaf_depth); dfree(c->d_leaf_far);
  c->have_dm = false;
}
static void free_weights(sand_ctx* c) {
  dfree(c->d_tables); dfree(c->d_pair_tables); dfree(c->d_w1_image); dfree(c->d_wimage); dfree(c->d_wimage_pair); dfree(c->d_tc4_w1); dfree(c->d_tc4_image); dfree(c->d_whidden); dfree(c->d_wt_f32);
  dfree(c->d_x3_image); dfree(c->d_x3_tables); c->have_x3 = false;
  c->have_w = false;
}
static void free_hostpipe(sand_ctx* c) {
  for (int i = 0; i < 2; ++i) {
    dfree(c->d_hpts[i]); dfree(c->d_hsdf[i]); dfree(c->d_hdep[i]);
    if (c->e_in[i]) cudaEventDestroy(c->e_in[i]);
    if (c->e_done[i]) cudaEventDestroy(c->e_done[i]);
    if (c->e_out[i]) cudaEventDestroy(c->e_out[i]);
    c->e_in[i] = c->e_done[i] = c->e_out[i] = nullptr;
  }
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  if (c->s_cmp) cudaStreamDestroy(c->s_cmp);
  c->s_h2d = c->s_d2h = c->s_cmp = nullptr;
  c->cap_h = 0;
}

extern "C" int sand_destroy(sand_ctx* ctx) {
  if (!ctx) return SAND_OK;
  cudaSetDevice(ctx->cfg.device);
  cudaStreamSynchronize(ctx->stream);
  cudaDeviceSynchronize();
  free_workspace(ctx);
  free_depthmap(ctx);
  free_weights(ctx);
  free_hostpipe(ctx);
  dfree(ctx->d_dp_tmp);
  dfree(ctx->d_dyn_h);
  dfree(ctx->d_axis); dfree(ctx->d_mpts); dfree(ctx->d_msdf); dfree(ctx->d_mdep); dfree(ctx->d_tricount); dfree(ctx->d_msigns);
  for (auto& q : ctx->evq)
    for (auto& v : q)
      if (v) cudaEventDestroy(v);
  delete ctx;
  return SAND_OK;
}

// ------------------------------------------------------------------------------- weights
static inline uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));  // inf/nan
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

extern "C" int sand_load_weights(sand_ctx* ctx, const float* blob, size_t n_floats) {
  if (!ctx || !blob) return fail(ctx, SAND_ERR_ARG, "sand_load_weights: NULL argument");
  const int L = ctx->cfg.L, H = ctx->cfg.H, tail = ctx->cfg.tail;
  const float w0 = ctx->cfg.omega0;
  size_t need = 3ull * H + H + (size_t)(L - 1) * ((size_t)H * H + H);
  need += (tail == SAND_TAIL_LINEAR) ? (size_t)L * (H + 1) : (size_t)(H + 1) + (size_t)(L - 1) * 2 * (H + 1);
  if (n_floats != need) return fail(ctx, SAND_ERR_SIZE, "weight blob has %zu floats, expected %zu", n_floats, need);
  CU(cudaSetDevice(ctx->cfg.device));
  // ---- parse canonical order
  std::vector<const float*> W(L), b(L), a(L), a1(L, nullptr);
  std::vector<float> c(L, 0.f), c1(L, 0.f);
  size_t o = 0;
  for (int i = 0; i < L; ++i) {
    const int fi = i == 0 ? 3 : H;
    W[i] = blob + o; o += (size_t)H * fi;
    b[i] = blob + o; o += H;
  }
  if (tail == SAND_TAIL_LINEAR) {
    for (int i = 0; i < L; ++i) { a[i] = blob + o; o += H; c[i] = blob[o++]; }
  } else {
    a[0] = blob + o; o += H; c[0] = blob[o++];
    for (int i = 1; i < L; ++i) {
      a[i] = blob + o; o += H; c[i] = blob[o++];
      a1[i] = blob + o; o += H; c1[i] = blob[o++];
    }
  }
  // ---- FP32 tables (layout documented in sand_internal.h MlpDev)
  MlpDev m{};
  m.L = L; m.H = H; m.tail = tail; m.omega0 = w0;
  // every per-layer row starts on a 16-byte boundary (H % 16 == 0): float4 table loads
  m.off_w1 = 0;
  m.off_bias = 4ll * H;
  m.off_a = m.off_bias + (long long)(L - 1) * H;
  m.off_a1 = m.off_a + (long long)L * H;
  m.off_c = m.off_a1 + (tail == SAND_TAIL_MULT ? (long long)(L - 1) * H : 0);
  m.off_c1 = m.off_c + L;
  long long ntab = m.off_c1 + (tail == SAND_TAIL_MULT ? (L - 1) : 0);
  ntab = (ntab + 3) & ~3ll;
  m.tables_floats = ntab;
  std::vector<float> tab((size_t)ntab, 0.f);
  for (int j = 0; j < H; ++j) {
    tab[4 * j + 0] = w0 * W[0][3 * j + 0];
    tab[4 * j + 1] = w0 * W[0][3 * j + 1];
    tab[4 * j + 2] = w0 * W[0][3 * j + 2];
    tab[4 * j + 3] = w0 * b[0][j];
  }
  for (int i = 1; i < L; ++i)
    for (int j = 0; j < H; ++j) tab[m.off_bias + (size_t)(i - 1) * H + j] = w0 * b[i][j];
  for (int i = 0; i < L; ++i) {
    std::memcpy(&tab[m.off_a + (size_t)i * H], a[i], sizeof(float) * H);
    tab[m.off_c + i] = c[i];
  }
  if (tail == SAND_TAIL_MULT)
    for (int i = 1; i < L; ++i) {
      std::memcpy(&tab[m.off_a1 + (size_t)(i - 1) * H], a1[i], sizeof(float) * H);
      tab[m.off_c1 + (i - 1)] = c1[i];
    }
  free_weights(ctx);
  CU(cudaMalloc(&ctx->d_tables, sizeof(float) * ntab));
  CU(cudaMemcpy(ctx->d_tables, tab.data(), sizeof(float) * ntab, cudaMemcpyHostToDevice));
  m.tables = ctx->d_tables;
  std::vector<uint8_t> pair_img;   // CTA-pair hidden-layer image (uploaded below)
  if (ctx->cfg.prec == SAND_BF16 && tc2_available(H)) {
    // CTA-pair kernel: w0 and the biases folded into split-BF16 MMA operands (tmlp_tc2.cu)
    std::vector<float> pt;
    std::vector<uint16_t> w1img;
    tc2_build_host(L, H, tail, w0, W.data(), b.data(), a.data(), a1.data(), c.data(), c1.data(), &m, &pt, &w1img,
                   &pair_img);
    CU(cudaMalloc(&ctx->d_w1_image, w1img.size() * 2));
    CU(cudaMemcpy(ctx->d_w1_image, w1img.data(), w1img.size() * 2, cudaMemcpyHostToDevice));
    m.w1_image = ctx->d_w1_image;
    CU(cudaMalloc(&ctx->d_pair_tables, sizeof(float) * pt.size()));
    CU(cudaMemcpy(ctx->d_pair_tables, pt.data(), sizeof(float) * pt.size(), cudaMemcpyHostToDevice));
    m.pair_tables = ctx->d_pair_tables;
  }
  if (ctx->cfg.prec == SAND_BF16 && tc4_available(H, tail)) {
    // slot-team CTA-pair kernel: its own layer-1 and hidden-layer images (tables shared with tmlp_tc2.cu)
    std::vector<uint16_t> w1img;
    std::vector<uint8_t> img;
    tc4_build_host(L, H, w0, W.data(), b.data(), &w1img, &img);
    dfree(ctx->d_tc4_w1);
    dfree(ctx->d_tc4_image);
    CU(cudaMalloc(&ctx->d_tc4_w1, w1img.size() * 2));
    CU(cudaMemcpy(ctx->d_tc4_w1, w1img.data(), w1img.size() * 2, cudaMemcpyHostToDevice));
    m.tc4_w1 = ctx->d_tc4_w1;
    if (!img.empty()) {
      CU(cudaMalloc(&ctx->d_tc4_image, img.size()));
      CU(cudaMemcpy(ctx->d_tc4_image, img.data(), img.size(), cudaMemcpyHostToDevice));
    }
    m.tc4_image = ctx->d_tc4_image;
  }
  if (ctx->cfg.prec == SAND_BF16 && tc3_available(H, tail)) {
    // wide CTA-pair kernel: padded-width tables, layer-1 and hidden-layer images (tmlp_tc3.cu)
    std::vector<float> pt;
    std::vector<uint16_t> w1img;
    std::vector<uint8_t> wimg;
    tc3_build_host(L, H, w0, W.data(), b.data(), a.data(), c.data(), &m, &pt, &w1img, &wimg);
    CU(cudaMalloc(&ctx->d_pair_tables, sizeof(float) * pt.size()));
    CU(cudaMemcpy(ctx->d_pair_tables, pt.data(), sizeof(float) * pt.size(), cudaMemcpyHostToDevice));
    m.pair_tables = ctx->d_pair_tables;
    CU(cudaMalloc(&ctx->d_w1_image, w1img.size() * 2));
    CU(cudaMemcpy(ctx->d_w1_image, w1img.data(), w1img.size() * 2, cudaMemcpyHostToDevice));
    m.w1_image = ctx->d_w1_image;
    if (!wimg.empty()) {
      CU(cudaMalloc(&ctx->d_wimage_pair, wimg.size()));
      CU(cudaMemcpy(ctx->d_wimage_pair, wimg.data(), wimg.size(), cudaMemcpyHostToDevice));
    }
  }
  if (L >= 2) {
    if (ctx->cfg.prec == SAND_FP32) {
      std::vector<float> wh((size_t)(L - 1) * H * H);
      for (int i = 1; i < L; ++i) std::memcpy(&wh[(size_t)(i - 1) * H * H], W[i], sizeof(float) * H * H);
      CU(cudaMalloc(&ctx->d_whidden, sizeof(float) * wh.size()));
      CU(cudaMemcpy(ctx->d_whidden, wh.data(), sizeof(float) * wh.size(), cudaMemcpyHostToDevice));
    } else {
      // BF16 image: [L-1][KC][H rows][128 B], SW128 K-major (element (n,k) of chunk kc at
      // (n/8)*1024 + (n%8)*128 + ((((k%64)/8) ^ (n%8)) * 16) + (k%8)*2; zero beyond K = H).
      const int KC = (H + 63) / 64;
      const size_t chunk = (size_t)H * 128;
      std::vector<uint16_t> img((size_t)(L - 1) * KC * chunk / 2, 0);
      for (int i = 1; i < L; ++i)
        for (int kc = 0; kc < KC; ++kc) {
          uint8_t* cb = reinterpret_cast<uint8_t*>(img.data()) + ((size_t)(i - 1) * KC + kc) * chunk;
          for (int n = 0; n < H; ++n)
            for (int kk = 0; kk < 64; ++kk) {
              const int k = 64 * kc + kk;
              if (k >= H) continue;
              const size_t byte = (size_t)(n / 8) * 1024 + (n % 8) * 128 + ((((kk / 8) ^ (n % 8)) * 16)) + (kk % 8) * 2;
              *reinterpret_cast<uint16_t*>(cb + byte) = bf16_rne(W[i][(size_t)n * H + k]);
            }
        }
      CU(cudaMalloc(&ctx->d_wimage, img.size() * 2));
      CU(cudaMemcpy(ctx->d_wimage, img.data(), img.size() * 2, cudaMemcpyHostToDevice));
      if (!pair_img.empty()) {
        CU(cudaMalloc(&ctx->d_wimage_pair, pair_img.size()));
        CU(cudaMemcpy(ctx->d_wimage_pair, pair_img.data(), pair_img.size(), cudaMemcpyHostToDevice));
      }
    }
  }
  if (x3_available(H)) {
    // split-FP16 x3 kernel (F16X3 queries and the FP32-accurate Eq. 5 population on tensor cores)
    std::vector<float> xt;
    std::vector<uint8_t> ximg;
    x3_build_host(L, H, tail, w0, W.data(), b.data(), a.data(), a1.data(), c.data(), c1.data(), &m, &xt, &ximg);
    CU(cudaMalloc(&ctx->d_x3_tables, sizeof(float) * xt.size()));
    CU(cudaMemcpy(ctx->d_x3_tables, xt.data(), sizeof(float) * xt.size(), cudaMemcpyHostToDevice));
    m.x3_tables = ctx->d_x3_tables;
    if (!ximg.empty()) {
      CU(cudaMalloc(&ctx->d_x3_image, ximg.size()));
      CU(cudaMemcpy(ctx->d_x3_image, ximg.data(), ximg.size(), cudaMemcpyHostToDevice));
    }
    m.x3_image = ctx->d_x3_image;
    ctx->have_x3 = true;
  }
  if (L >= 2) {
    // FP32 W^T for the depth-map population kernels (Eq. 5 needs FP32 whatever the query precision)
    std::vector<float> wt((size_t)(L - 1) * H * H);
    for (int i = 1; i < L; ++i)
      for (int j = 0; j < H; ++j)
        for (int k = 0; k < H; ++k) wt[(size_t)(i - 1) * H * H + (size_t)k * H + j] = W[i][(size_t)j * H + k];
    CU(cudaMalloc(&ctx->d_wt_f32, sizeof(float) * wt.size()));
    CU(cudaMemcpy(ctx->d_wt_f32, wt.data(), sizeof(float) * wt.size(), cudaMemcpyHostToDevice));
  }
  m.w_hidden = ctx->d_whidden;
  m.w_image = ctx->d_wimage;
  m.w_image_pair = ctx->d_wimage_pair;
  m.kprof = ctx->kprof;
  ctx->mlp = m;
  ctx->have_w = true;
  return SAND_OK;
}

// ------------------------------------------------------------------------------- depth map
extern "C" int sand_load_depthmap(sand_ctx* ctx, const sand_depthmap* dm) {
  if (!ctx || !dm || !dm->depth) return fail(ctx, SAND_ERR_ARG, "sand_load_depthmap: NULL argument");
  CU(cudaSetDevice(ctx->cfg.device));
  const int L = ctx->cfg.L;
  LookupParams lp{};
  lp.L = L;
  lp.level = dm->level;
  if (dm->kind == 0) {
    if (dm->level < 0 || dm->level > 10) return fail(ctx, SAND_ERR_DEPTHMAP, "voxel level %d outside [0,10]", dm->level);
    const size_t nc = (size_t)1 << (3 * dm->level);
    bool far_needed = false;
    for (size_t i = 0; i < nc; ++i) {
      if (dm->depth[i] > L) return fail(ctx, SAND_ERR_DEPTHMAP, "voxel %zu has depth %d > L = %d", i, dm->depth[i], L);
      far_needed |= dm->depth[i] == 0;
    }
    if (far_needed && !dm->far_sdf) return fail(ctx, SAND_ERR_DEPTHMAP, "depth-0 voxels need far_sdf");
    free_depthmap(ctx);
    CU(cudaMalloc(&ctx->d_grid, nc));
    CU(cudaMemcpy(ctx->d_grid, dm->depth, nc, cudaMemcpyHostToDevice));
    if (dm->far_sdf) {
      CU(cudaMalloc(&ctx->d_grid_far, nc * 4));
      CU(cudaMemcpy(ctx->d_grid_far, dm->far_sdf, nc * 4, cudaMemcpyHostToDevice));
    }
    lp.dense = 1;
  } else if (dm->kind == 1) {
    if (!dm->nodes || dm->n_nodes < 1 || dm->n_leaves < 1)
      return fail(ctx, SAND_ERR_ARG, "octree needs nodes, n_nodes >= 1, n_leaves >= 1");
    if (dm->level < 0 || dm->level > 20) return fail(ctx, SAND_ERR_DEPTHMAP, "octree level %d outside [0,20]", dm->level);
    if (dm->n_nodes >= (1ll << 31) || dm->n_leaves >= (1ll << 31)) return fail(ctx, SAND_ERR_DEPTHMAP, "octree too large");
    bool far_needed = false;
    for (long long i = 0; i < dm->n_leaves; ++i) {
      if (dm->depth[i] > L) return fail(ctx, SAND_ERR_DEPTHMAP, "leaf %lld has depth %d > L = %d", i, dm->depth[i], L);
      far_needed |= dm->depth[i] == 0;
    }
    if (far_needed && !dm->far_sdf) return fail(ctx, SAND_ERR_DEPTHMAP, "depth-0 leaves need far_sdf");
    // structural validation: BFS from the root, every internal node's 8 children in range, every
    // node reached at most once (acyclic tree), descent depth <= level.
    std::vector<uint8_t> seen((size_t)dm->n_nodes, 0);
    std::vector<std::pair<uint32_t, int>> q;
    q.push_back({0u, 0});
    seen[0] = 1;
    for (size_t h = 0; h < q.size(); ++h) {
      const uint32_t v = dm->nodes[q[h].first];
      const int lev = q[h].second;
      if (v >> 31) {
        if ((long long)(v & 0x7FFFFFFFu) >= dm->n_leaves) return fail(ctx, SAND_ERR_DEPTHMAP, "leaf index out of range");
        continue;
      }
      if (lev >= dm->level) return fail(ctx, SAND_ERR_DEPTHMAP, "octree deeper than level %d", dm->level);
      if ((long long)v + 8 > dm->n_nodes) return fail(ctx, SAND_ERR_DEPTHMAP, "child index out of range");
      for (uint32_t o = 0; o < 8; ++o) {
        if (seen[v + o]) return fail(ctx, SAND_ERR_DEPTHMAP, "node %u reached twice (not a tree)", v + o);
        seen[v + o] = 1;
        q.push_back({v + o, lev + 1});
      }
    }
    free_depthmap(ctx);
    CU(cudaMalloc(&ctx->d_nodes, dm->n_nodes * 4));
    CU(cudaMemcpy(ctx->d_nodes, dm->nodes, dm->n_nodes * 4, cudaMemcpyHostToDevice));
    CU(cudaMalloc(&ctx->d_leaf_depth, dm->n_leaves));
    CU(cudaMemcpy(ctx->d_leaf_depth, dm->depth, dm->n_leaves, cudaMemcpyHostToDevice));
    if (dm->far_sdf) {
      CU(cudaMalloc(&ctx->d_leaf_far, dm->n_leaves * 4));
      CU(cudaMemcpy(ctx->d_leaf_far, dm->far_sdf, dm->n_leaves * 4, cudaMemcpyHostToDevice));
    }
    lp.nodes = ctx->d_nodes;
    lp.leaf_depth = ctx->d_leaf_depth;
    lp.leaf_far = ctx->d_leaf_far;
    lp.dense = 0;
    if (dm->level <= 8) {
      // bake to a dense 2^level grid: one load per query instead of a pointer-chasing descent
      const size_t nc = (size_t)1 << (3 * dm->level);
      CU(cudaMalloc(&ctx->d_grid, nc));
      if (dm->far_sdf) CU(cudaMalloc(&ctx->d_grid_far, nc * 4));
      struct DevFlag {   // freed on every return path
        int* p = nullptr;
        ~DevFlag() { if (p) cudaFree(p); }
      } err;
      CU(cudaMalloc(&err.p, 4));
      CU(cudaMemset(err.p, 0, 4));
      CU(launch_bake_octree(ctx->d_nodes, ctx->d_leaf_depth, ctx->d_leaf_far, dm->level, ctx->d_grid,
                            ctx->d_grid_far, err.p, ctx->stream));
      int herr = 0;
      CU(cudaMemcpyAsync(&herr, err.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      if (herr) return fail(ctx, SAND_ERR_DEPTHMAP, "octree bake failed (descent exceeded level)");
      lp.dense = 1;
    } else {
      // deeper octrees keep the descent, started from a dense table of the level-7 nodes (8 MB)
      lp.top_level = 7;
      CU(cudaMalloc(&ctx->d_top, sizeof(uint32_t) << (3 * lp.top_level)));
      CU(launch_bake_top(ctx->d_nodes, lp.top_level, ctx->d_top, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      lp.top = ctx->d_top;
    }
  } else {
    return fail(ctx, SAND_ERR_ARG, "depth map kind %d (0 = voxel, 1 = octree)", dm->kind);
  }
  lp.grid = ctx->d_grid;
  lp.grid_far = ctx->d_grid_far;
  ctx->lp = lp;
  ctx->have_dm = true;
  return SAND_OK;
}

extern "C" int sand_set_stream(sand_ctx* ctx, void* s) {
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  ctx->stream = reinterpret_cast<cudaStream_t>(s);
  return SAND_OK;
}

// Eq. 5 population on the split-FP16 tensor-core kernel when the width and shared memory allow it
static bool use_x3_population(const sand_ctx* ctx) {
  return ctx->fp32_tensor && ctx->have_x3 && x3_usable(ctx->cfg.L, ctx->cfg.H, ctx->cfg.tail, 1);
}

extern "C" int sand_set_option(sand_ctx* ctx, int option, int64_t value) {
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  switch (option) {
    case SAND_OPT_PAIR_KERNEL:
      if (value < 0 || value > 2) return fail(ctx, SAND_ERR_ARG, "SAND_OPT_PAIR_KERNEL takes 0, 1 or 2");
      if (value >= 1 && !ctx->pair_ok) return fail(ctx, SAND_ERR_UNSUPPORTED, "no CTA-pair kernel for this (prec, L, H, tail)");
      if (value == 2 && !ctx->team_ok) return fail(ctx, SAND_ERR_UNSUPPORTED, "no slot-team CTA-pair kernel for this (prec, L, H, tail)");
      ctx->use_pair = (int)value;
      return SAND_OK;
    case SAND_OPT_DYN_SCHEDULE:
      if (value < 0 || value > 2) return fail(ctx, SAND_ERR_ARG, "SAND_OPT_DYN_SCHEDULE takes 0, 1 or 2");
      ctx->dyn_schedule = (int)value;
      return SAND_OK;
    case SAND_OPT_FP32_TENSOR:
      if (value != 0 && value != 1) return fail(ctx, SAND_ERR_ARG, "SAND_OPT_FP32_TENSOR takes 0 or 1");
      ctx->fp32_tensor = (int)value;
      return SAND_OK;
    case SAND_OPT_KPROF:
      if (value < 0 || value > 3) return fail(ctx, SAND_ERR_ARG, "SAND_OPT_KPROF takes 0..3");
      ctx->kprof = (int)value;
      ctx->mlp.kprof = (int)value;
      return SAND_OK;
    default:
      return fail(ctx, SAND_ERR_ARG, "unknown option %d", option);
  }
}

extern "C" int sand_get_option(const sand_ctx* ctx, int option, int64_t* value) {
  if (!ctx || !value) return SAND_ERR_ARG;
  switch (option) {
    case SAND_OPT_PAIR_KERNEL: *value = ctx->use_pair; return SAND_OK;
    case SAND_OPT_DYN_SCHEDULE: *value = ctx->dyn_schedule; return SAND_OK;
    case SAND_OPT_KPROF: *value = ctx->kprof; return SAND_OK;
    case SAND_OPT_FP32_TENSOR: *value = ctx->fp32_tensor; return SAND_OK;
    default: return SAND_ERR_ARG;
  }
}

extern "C" int sand_set_lod_cap(sand_ctx* ctx, int cap) {
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (cap < 1 || cap > ctx->cfg.L) return fail(ctx, SAND_ERR_ARG, "lod cap %d outside [1,%d]", cap, ctx->cfg.L);
  ctx->lod_cap = cap;
  return SAND_OK;
}

static int ensure_workspace(sand_ctx* ctx, long long n) {
  const long long nblk = (n + kLookupChunk - 1) / kLookupChunk;
  if (n <= ctx->cap_n && nblk <= ctx->cap_nblk) return SAND_OK;
  CU(cudaStreamSynchronize(ctx->stream));
  free_workspace(ctx);
  CU(cudaMalloc(&ctx->d_hist, sizeof(uint32_t) * (size_t)nblk * kMaxBins));
  CU(cudaMalloc(&ctx->d_offs, sizeof(uint32_t) * (size_t)nblk * kMaxBins));
  CU(cudaMalloc(&ctx->d_scan, sizeof(unsigned long long) * (size_t)scan_scratch_words(nblk)));
  CU(cudaMalloc(&ctx->d_perm, sizeof(uint32_t) * (size_t)std::max(n, 1ll)));
  CU(cudaMalloc(&ctx->d_meta, sizeof(QueryMeta)));
  ctx->cap_n = n;
  ctx->cap_nblk = nblk;
  return SAND_OK;
}

extern "C" int sand_reserve(sand_ctx* ctx, int64_t n_max) {
  if (!ctx || n_max < 0) return fail(ctx, SAND_ERR_ARG, "sand_reserve: bad argument");
  CU(cudaSetDevice(ctx->cfg.device));
  return ensure_workspace(ctx, n_max);
}

extern "C" int sand_query(sand_ctx* ctx, const float* d_points, int64_t n, float* d_sdf, uint8_t* d_depth) {
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (n < 0) return fail(ctx, SAND_ERR_ARG, "n < 0");
  if (!ctx->have_w || !ctx->have_dm) return fail(ctx, SAND_ERR_STATE, "load weights and depth map before sand_query");
  if (n == 0) return SAND_OK;
  if (!d_points || !d_sdf || !d_depth) return fail(ctx, SAND_ERR_ARG, "NULL buffer");
  if ((reinterpret_cast<uintptr_t>(d_points) & 3) || (reinterpret_cast<uintptr_t>(d_sdf) & 3))
    return fail(ctx, SAND_ERR_ARG, "points/sdf must be 4-byte aligned");
  if (n >= (1ll << 32) - 1) return fail(ctx, SAND_ERR_ARG, "n = %lld exceeds 2^32-2 points per query", (long long)n);
  CU(cudaSetDevice(ctx->cfg.device));
  int rc = ensure_workspace(ctx, n);
  if (rc) return rc;
  const long long nblk = (n + kLookupChunk - 1) / kLookupChunk;
  LookupParams lp = ctx->lp;
  lp.cap = ctx->lod_cap;
  cudaStream_t st = ctx->stream;
  if (ctx->nq == 1024) ctx->nq = 0;  // bounded: sums cover at most the last 1024 queries
  if (ctx->nq == ctx->evq.size()) {
    std::array<cudaEvent_t, 4> q{};
    for (auto& v : q) CU(cudaEventCreate(&v));
    ctx->evq.push_back(q);
  }
  const size_t qi = ctx->nq++;
  cudaEvent_t* ev = ctx->evq[qi].data();
  NvtxRange nq("sand_query");
  CU(cudaEventRecord(ev[0], st));
  {
    NvtxRange r("K1 depth-map lookup");
    CU(launch_lookup(d_points, n, lp, d_depth, d_sdf, ctx->d_hist, nblk, st));
  }
  CU(cudaEventRecord(ev[1], st));
  {
    NvtxRange r("K2 binning (scan + scatter)");
    CU(launch_scan(ctx->d_hist, nblk, ctx->cfg.L, tmlp_tile_rows(ctx->cfg.H, ctx->cfg.prec, ctx->use_pair),
                   tc4_runs(ctx->cfg.L, ctx->cfg.H, ctx->cfg.tail, ctx->cfg.prec, ctx->use_pair) ? 1 : 0, ctx->d_offs,
                   ctx->d_meta, ctx->d_scan, st));
    CU(launch_scatter(d_depth, n, ctx->cfg.L, ctx->d_offs, ctx->d_perm, nblk, st));
  }
  CU(cudaEventRecord(ev[2], st));
  NvtxRange r3("K3 T-MLP");
  if (ctx->cfg.prec == SAND_F16X3)
    CU(launch_tmlp_x3(ctx->mlp, d_points, ctx->d_perm, ctx->d_meta, d_sdf, ctx->num_sms, st));
  else if (ctx->cfg.prec == SAND_FP32 && !simt_supported_H(ctx->cfg.H))
    CU(launch_query_fp32(ctx->mlp, ctx->d_wt_f32, d_points, ctx->d_perm, ctx->d_meta, d_sdf, ctx->num_sms, st));
  else if (ctx->cfg.prec == SAND_FP32)
    CU(launch_tmlp_simt(ctx->mlp, d_points, ctx->d_perm, ctx->d_meta, d_sdf, ctx->num_sms, st));
  else
    CU(launch_tmlp_tc(ctx->mlp, d_points, ctx->d_perm, ctx->d_meta, d_sdf, ctx->num_sms, st, ctx->use_pair));
  CU(cudaEventRecord(ev[3], st));
  ctx->last_q = qi;
  ctx->have_stats = true;
  ctx->last_n = n;
  return SAND_OK;
}

static int ensure_hostpipe(sand_ctx* ctx, long long chunk) {
  if (chunk <= ctx->cap_h) return SAND_OK;
  free_hostpipe(ctx);
  for (int i = 0; i < 2; ++i) {
    CU(cudaMalloc(&ctx->d_hpts[i], sizeof(float) * 3 * (size_t)chunk));
    CU(cudaMalloc(&ctx->d_hsdf[i], sizeof(float) * (size_t)chunk));
    CU(cudaMalloc(&ctx->d_hdep[i], (size_t)chunk));
    CU(cudaEventCreateWithFlags(&ctx->e_in[i], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->e_done[i], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ctx->e_out[i], cudaEventDisableTiming));
  }
  CU(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&ctx->s_cmp, cudaStreamNonBlocking));
  ctx->cap_h = chunk;
  return SAND_OK;
}

extern "C" int sand_query_host(sand_ctx* ctx, const float* h_points, int64_t n, float* h_sdf, uint8_t* h_depth,
                               int64_t chunk_points) {
  NvtxRange nvtx_("sand_query_host (pipelined H2D / query / D2H)");
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (n < 0 || chunk_points < 0) return fail(ctx, SAND_ERR_ARG, "negative size");
  if (!ctx->have_w || !ctx->have_dm) return fail(ctx, SAND_ERR_STATE, "load weights and depth map first");
  if (n == 0) return SAND_OK;
  if (!h_points || !h_sdf || !h_depth) return fail(ctx, SAND_ERR_ARG, "NULL buffer");
  CU(cudaSetDevice(ctx->cfg.device));
  long long chunk = chunk_points;
  if (chunk == 0) chunk = std::min<long long>(std::max<long long>(n / 8, 1ll << 21), 1ll << 23);   // sand.h
  chunk = std::min<long long>(chunk, n);
  chunk = (chunk + 3) & ~3ll;
  int rc = ensure_hostpipe(ctx, chunk);
  if (rc) return rc;
  rc = ensure_workspace(ctx, chunk);
  if (rc) return rc;
  cudaStream_t user = ctx->stream;
  CU(cudaStreamSynchronize(user));
  ctx->stream = ctx->s_cmp;
  const long long nch = (n + chunk - 1) / chunk;
  int ret = SAND_OK;
  for (long long i = 0; i < nch && ret == SAND_OK; ++i) {
    const int b = (int)(i & 1);
    const long long p0 = i * chunk, m = std::min(chunk, n - p0);
    if (i >= 2) {
      // input buffer b is free once the query of chunk i-2 has finished
      if (cudaStreamWaitEvent(ctx->s_h2d, ctx->e_done[b], 0) != cudaSuccess) { ret = fail(ctx, SAND_ERR_CUDA, "wait"); break; }
      if (cudaStreamWaitEvent(ctx->s_cmp, ctx->e_out[b], 0) != cudaSuccess) { ret = fail(ctx, SAND_ERR_CUDA, "wait"); break; }
    }
    if (cudaMemcpyAsync(ctx->d_hpts[b], h_points + 3 * p0, sizeof(float) * 3 * m, cudaMemcpyHostToDevice, ctx->s_h2d) != cudaSuccess ||
        cudaEventRecord(ctx->e_in[b], ctx->s_h2d) != cudaSuccess ||
        cudaStreamWaitEvent(ctx->s_cmp, ctx->e_in[b], 0) != cudaSuccess) {
      ret = fail(ctx, SAND_ERR_CUDA, "host pipeline H2D failed");
      break;
    }
    ret = sand_query(ctx, ctx->d_hpts[b], m, ctx->d_hsdf[b], ctx->d_hdep[b]);
    if (ret) break;
    if (cudaEventRecord(ctx->e_done[b], ctx->s_cmp) != cudaSuccess ||
        cudaStreamWaitEvent(ctx->s_d2h, ctx->e_done[b], 0) != cudaSuccess ||
        cudaMemcpyAsync(h_sdf + p0, ctx->d_hsdf[b], sizeof(float) * m, cudaMemcpyDeviceToHost, ctx->s_d2h) != cudaSuccess ||
        cudaMemcpyAsync(h_depth + p0, ctx->d_hdep[b], (size_t)m, cudaMemcpyDeviceToHost, ctx->s_d2h) != cudaSuccess ||
        cudaEventRecord(ctx->e_out[b], ctx->s_d2h) != cudaSuccess) {
      ret = fail(ctx, SAND_ERR_CUDA, "host pipeline D2H failed");
      break;
    }
  }
  cudaError_t e1 = cudaStreamSynchronize(ctx->s_d2h);
  cudaError_t e2 = cudaStreamSynchronize(ctx->s_cmp);
  ctx->stream = user;
  if (ret) return ret;
  if (e1 != cudaSuccess || e2 != cudaSuccess)
    return fail(ctx, SAND_ERR_CUDA, "host pipeline: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  return SAND_OK;
}

extern "C" int sand_get_stats(sand_ctx* ctx, sand_stats* out) {
  if (!ctx || !out) return fail(ctx, SAND_ERR_ARG, "NULL argument");
  std::memset(out, 0, sizeof(*out));
  if (!ctx->have_stats) return SAND_OK;
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaStreamSynchronize(ctx->stream));
  QueryMeta m{};
  CU(cudaMemcpy(&m, ctx->d_meta, sizeof m, cudaMemcpyDeviceToHost));
  const int L = ctx->cfg.L, H = ctx->cfg.H;
  out->n = ctx->last_n;
  out->n_nonfinite = m.count[L + 1];
  for (int d = 0; d <= L; ++d) {
    out->per_depth[d] = m.count[d];
    if (d >= 1) {
      out->flops_exec += (double)m.count[d] * (d - 1) * 2.0 * H * H;
      out->flops_ns += (double)m.count[d] * d * 2.0 * H * H;
    }
  }
  out->tiles = m.total_tiles;
  for (size_t i = 0; i < ctx->nq; ++i) {
    cudaEvent_t* ev = ctx->evq[i].data();
    float a, b, c, t;
    CU(cudaEventElapsedTime(&a, ev[0], ev[1]));
    CU(cudaEventElapsedTime(&b, ev[1], ev[2]));
    CU(cudaEventElapsedTime(&c, ev[2], ev[3]));
    CU(cudaEventElapsedTime(&t, ev[0], ev[3]));
    out->ms_lookup_sum += a; out->ms_bin_sum += b; out->ms_mlp_sum += c; out->ms_total_sum += t;
    if (i == ctx->last_q) { out->ms_lookup = a; out->ms_bin = b; out->ms_mlp = c; out->ms_total = t; }
  }
  out->queries = (int64_t)ctx->nq;
  ctx->nq = 0;
  return SAND_OK;
}

// Diagnostic (not in sand.h's main path): copy the binning permutation of the last query to host.
extern "C" int sand_debug_perm(sand_ctx* ctx, uint32_t* host_perm, int64_t cap, int64_t* n_binned) {
  if (!ctx || !n_binned) return fail(ctx, SAND_ERR_ARG, "NULL argument");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaStreamSynchronize(ctx->stream));
  if (!ctx->have_stats) { *n_binned = 0; return SAND_OK; }
  QueryMeta m{};
  CU(cudaMemcpy(&m, ctx->d_meta, sizeof m, cudaMemcpyDeviceToHost));
  long long nb = 0;
  for (int d = 1; d <= ctx->cfg.L; ++d) nb += m.count[d];
  *n_binned = nb;
  if (host_perm && cap > 0) CU(cudaMemcpy(host_perm, ctx->d_perm, sizeof(uint32_t) * (size_t)std::min<long long>(cap, nb), cudaMemcpyDeviceToHost));
  return SAND_OK;
}

// ------------------------------------------------------------------------------- marching cubes
static int mesh_prepare(sand_ctx* ctx, int R, int planes) {
  CU(mc_upload_tables());
  const size_t nw = mc_sign_words(R, planes);
  if (nw > ctx->cap_msigns) {
    CU(cudaStreamSynchronize(ctx->stream));
    dfree(ctx->d_msigns);
    ctx->cap_msigns = 0;
    CU(cudaMalloc(&ctx->d_msigns, sizeof(uint32_t) * nw));
    ctx->cap_msigns = nw;
  }
  if (ctx->axis_R != R) {
    CU(cudaStreamSynchronize(ctx->stream));
    dfree(ctx->d_axis);
    CU(cudaMalloc(&ctx->d_axis, sizeof(float) * R));
    ctx->axis_R = R;
    CU(launch_grid_axis(R, ctx->d_axis, ctx->stream));
  }
  if (!ctx->d_tricount) CU(cudaMalloc(&ctx->d_tricount, mc_counter_words() * sizeof(unsigned long long)));
  CU(cudaMemsetAsync(ctx->d_tricount, 0, sizeof(unsigned long long), ctx->stream));
  return SAND_OK;
}

static int mesh_finish(sand_ctx* ctx, int64_t* n_tris) {
  unsigned long long h = 0;
  CU(cudaMemcpyAsync(&h, ctx->d_tricount, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  *n_tris = (int64_t)h;
  return SAND_OK;
}

extern "C" int sand_marching_cubes(sand_ctx* ctx, const float* d_sdf, int R, float* d_tris, int64_t cap,
                                   int64_t* n_tris) {
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (R < 2 || R > 65535 || cap < 0 || !n_tris || !d_sdf || (cap > 0 && !d_tris))
    return fail(ctx, SAND_ERR_ARG, "sand_marching_cubes: R outside [2, 65535], cap < 0 or NULL argument");
  CU(cudaSetDevice(ctx->cfg.device));
  int rc = mesh_prepare(ctx, R, R);
  if (rc) return rc;
  CU(launch_marching_cubes(d_sdf, R, 0, R - 1, 0, ctx->d_axis, d_tris, cap, ctx->d_tricount, ctx->d_msigns,
                           ctx->num_sms, ctx->stream));
  return mesh_finish(ctx, n_tris);
}

extern "C" int sand_mesh_grid(sand_ctx* ctx, int R, int slab, float* d_tris, int64_t cap, int64_t* n_tris) {
  NvtxRange nvtx_("sand_mesh_grid");
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (R < 2 || R > 65535 || slab < 0 || cap < 0 || !n_tris || (cap > 0 && !d_tris))
    return fail(ctx, SAND_ERR_ARG, "sand_mesh_grid: R outside [2, 65535], slab < 0, cap < 0 or NULL argument");
  if (!ctx->have_w || !ctx->have_dm) return fail(ctx, SAND_ERR_STATE, "load weights and depth map first");
  CU(cudaSetDevice(ctx->cfg.device));
  if (slab == 0) slab = 64;
  if (slab > R - 1) slab = R - 1;
  int rc = mesh_prepare(ctx, R, slab + 1);
  if (rc) return rc;
  const long long np = (long long)R * R * (slab + 1);   // points of the slab's slab + 1 planes
  if (np > ctx->cap_m) {
    CU(cudaStreamSynchronize(ctx->stream));
    dfree(ctx->d_mpts); dfree(ctx->d_msdf); dfree(ctx->d_mdep);
    CU(cudaMalloc(&ctx->d_mpts, sizeof(float) * 3 * np));
    CU(cudaMalloc(&ctx->d_msdf, sizeof(float) * np));
    CU(cudaMalloc(&ctx->d_mdep, (size_t)np));
    ctx->cap_m = np;
  }
  const long long R2 = (long long)R * R;
  for (int kc0 = 0; kc0 < R - 1; kc0 += slab) {
    const int kc1 = std::min(kc0 + slab, R - 1);   // cubes kc0 .. kc1 - 1 need planes kc0 .. kc1
    // plane kc0 was the previous slab's last plane: move its sdf down instead of querying it again
    const int q0 = kc0 == 0 ? 0 : 1;
    if (q0) CU(cudaMemcpyAsync(ctx->d_msdf, ctx->d_msdf + (long long)slab * R2, sizeof(float) * R2,
                               cudaMemcpyDeviceToDevice, ctx->stream));
    const int npl = kc1 - kc0 + 1 - q0;
    const long long n = R2 * npl;
    CU(launch_grid_points(ctx->d_axis, R, kc0 + q0, npl, ctx->d_mpts, ctx->num_sms, ctx->stream));
    rc = sand_query(ctx, ctx->d_mpts, n, ctx->d_msdf + q0 * R2, ctx->d_mdep);
    if (rc) return rc;
    CU(launch_marching_cubes(ctx->d_msdf, R, kc0, kc1, kc0, ctx->d_axis, d_tris, cap, ctx->d_tricount,
                             ctx->d_msigns, ctx->num_sms, ctx->stream));
  }
  return mesh_finish(ctx, n_tris);
}

// ------------------------------------------------------------------------------- depth-map population
extern "C" int sand_required_depth(sand_ctx* ctx, const float* d_points, int64_t n, float r, int near,
                                   uint8_t* d_out_depth) {
  NvtxRange nvtx_("sand_required_depth (Eq. 5)");
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (n < 0 || !(r >= 0.0f)) return fail(ctx, SAND_ERR_ARG, "sand_required_depth: n < 0 or r < 0");
  if (!ctx->have_w) return fail(ctx, SAND_ERR_STATE, "load weights before sand_required_depth");
  if (n == 0) return SAND_OK;
  if (!d_points || !d_out_depth) return fail(ctx, SAND_ERR_ARG, "NULL buffer");
  if (!depthpop_supported(ctx->cfg.H)) return fail(ctx, SAND_ERR_UNSUPPORTED, "H = %d", ctx->cfg.H);
  CU(cudaSetDevice(ctx->cfg.device));
  if (use_x3_population(ctx))
    CU(launch_required_depth_x3(ctx->mlp, d_points, n, r, near ? 1 : 0, d_out_depth, ctx->num_sms, ctx->stream));
  else
    CU(launch_required_depth(ctx->mlp, ctx->d_wt_f32, d_points, n, r, near ? 1 : 0, d_out_depth, ctx->num_sms,
                             ctx->stream));
  return SAND_OK;
}

extern "C" int sand_query_dynamic(sand_ctx* ctx, const float* d_points, int64_t n, float r, float* d_out_sdf,
                                  uint8_t* d_out_exit_depth) {
  NvtxRange nvtx_("sand_query_dynamic");
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (n < 0 || !(r >= 0.0f)) return fail(ctx, SAND_ERR_ARG, "sand_query_dynamic: n < 0 or r < 0");
  if (!ctx->have_w) return fail(ctx, SAND_ERR_STATE, "load weights before sand_query_dynamic");
  if (n == 0) return SAND_OK;
  if (!d_points || !d_out_sdf || !d_out_exit_depth) return fail(ctx, SAND_ERR_ARG, "NULL buffer");
  if (!depthpop_supported(ctx->cfg.H)) return fail(ctx, SAND_ERR_UNSUPPORTED, "H = %d", ctx->cfg.H);
  CU(cudaSetDevice(ctx->cfg.device));
  // SAND_OPT_DYN_SCHEDULE: 0 = tile-level early exit, 1 = pools re-compacted after every layer (FP32 SIMT),
  // 2 = full-depth split-FP16 tensor evaluation with the exit layer selected per point (H in {64, 128, 256})
  if (ctx->dyn_schedule == 2) {
    if (!(ctx->have_x3 && x3_usable(ctx->cfg.L, ctx->cfg.H, ctx->cfg.tail, 2)))
      return fail(ctx, SAND_ERR_UNSUPPORTED, "SAND_OPT_DYN_SCHEDULE = 2 needs H in {64, 128, 256}");
    CU(launch_query_dynamic_x3(ctx->mlp, d_points, n, r, d_out_sdf, d_out_exit_depth, ctx->num_sms, ctx->stream));
    return SAND_OK;
  }
  const bool pool = ctx->dyn_schedule == 1;
  float* hbuf = nullptr;
  if (pool) {
    if (!ctx->d_dyn_h) {
      CU(cudaMalloc(&ctx->d_dyn_h, sizeof(float) * dynamic_scratch_floats(ctx->cfg.H, ctx->num_sms)));
    }
    hbuf = ctx->d_dyn_h;
  }
  CU(launch_query_dynamic(ctx->mlp, ctx->d_wt_f32, d_points, n, r, d_out_sdf, d_out_exit_depth, hbuf, ctx->num_sms,
                          ctx->stream));
  return SAND_OK;
}

extern "C" int sand_populate_leaf_depths(sand_ctx* ctx, const float* d_samples, int64_t n_leaves,
                                         int samples_per_leaf, float r, uint8_t* d_leaf_depth) {
  NvtxRange nvtx_("sand_populate_leaf_depths (Eq. 5/6)");
  if (!ctx) return fail(ctx, SAND_ERR_ARG, "NULL ctx");
  if (n_leaves < 0 || samples_per_leaf < 1 || !(r >= 0.0f))
    return fail(ctx, SAND_ERR_ARG, "sand_populate_leaf_depths: bad size or r");
  if (!ctx->have_w) return fail(ctx, SAND_ERR_STATE, "load weights before sand_populate_leaf_depths");
  if (n_leaves == 0) return SAND_OK;
  if (!d_samples || !d_leaf_depth) return fail(ctx, SAND_ERR_ARG, "NULL buffer");
  if (!depthpop_supported(ctx->cfg.H)) return fail(ctx, SAND_ERR_UNSUPPORTED, "H = %d", ctx->cfg.H);
  CU(cudaSetDevice(ctx->cfg.device));
  const long long ns = n_leaves * (long long)samples_per_leaf;
  if (ns > ctx->cap_dp) {
    CU(cudaStreamSynchronize(ctx->stream));
    dfree(ctx->d_dp_tmp);
    CU(cudaMalloc(&ctx->d_dp_tmp, (size_t)ns));
    ctx->cap_dp = ns;
  }
  if (use_x3_population(ctx))
    CU(launch_required_depth_x3(ctx->mlp, d_samples, ns, r, 1, ctx->d_dp_tmp, ctx->num_sms, ctx->stream));
  else
    CU(launch_required_depth(ctx->mlp, ctx->d_wt_f32, d_samples, ns, r, 1, ctx->d_dp_tmp, ctx->num_sms, ctx->stream));
  CU(launch_leaf_max(ctx->d_dp_tmp, n_leaves, samples_per_leaf, d_leaf_depth, ctx->stream));
  return SAND_OK;
}
