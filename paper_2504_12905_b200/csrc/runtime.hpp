// runtime.hpp — host-side C++ runtime of libslm_b200 (compiled with g++;
// the kernels it drives live in the *.cu files).
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "layout.hpp"

namespace slm {

struct CudaError : std::runtime_error {
    cudaError_t code;
    CudaError(cudaError_t c, const char* what, const char* file, int line)
        : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(c) + " at " + file + ":" +
                             std::to_string(line) + " (" + what + ")"),
          code(c) {}
};

#define SLM_CUDA_CHECK(x)                                                          \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) throw ::slm::CudaError(e_, #x, __FILE__, __LINE__); \
    } while (0)

extern std::atomic<long long> g_launches;  // kernels launched by this library

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // Grow-only allocation with 25% headroom (sizes such as the tile-list length
    // drift from one LM step to the next; cudaFree/cudaMalloc synchronise the
    // device); contents are undefined after a reallocation.
    T* ensure(size_t count) {
        if (count <= n && p) return p;
        release();
        const size_t cap = count + count / 4;
        const size_t bytes = (cap > 0 ? cap : 1) * sizeof(T);
        SLM_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&p), bytes));
        n = cap;
        return p;
    }
    T* ensure_zero(size_t count, cudaStream_t st) {
        const bool fresh = count > n || !p;
        ensure(count);
        if (fresh) SLM_CUDA_CHECK(cudaMemsetAsync(p, 0, (n > 0 ? n : 1) * sizeof(T), st));
        return p;
    }
};

// ---- launchers (defined in the .cu files)
void launch_prepare(const double* beta, int G, int Gp, const DevCam* cams, int V, float4* rec,
                    unsigned long long* keys, short4* rect, unsigned long long* n_entries, int* err,
                    double* rec64, float4* conic, cudaStream_t st);
void launch_depth_init(const unsigned long long* keys, const short4* rect, int G, int Gp, int V,
                       unsigned long long* kout, unsigned* vout, unsigned long long* and_or, cudaStream_t st);
void build_tile_lists(const unsigned long long* keys, const short4* rect, const DevCam* cams, int G, int Gp, int V,
                      int n_tiles, long long n_entries, unsigned long long and_k, unsigned long long or_k,
                      const TileSortBuffers& b, int* entries, int* tile_offsets, cudaStream_t st);
long long radix_hist_size(long long n);
long long scan_scratch(long long n);
void launch_apply_update(double* beta, const float* delta, int G, int Gp, double eta, float* beta32,
                         cudaStream_t st);
void launch_apply_update_f64(double* beta, const double* delta_aos, int G, int Gp, double eta,
                             float* beta32, cudaStream_t st);
void launch_beta_mirror(const double* beta, float* beta32, int n, cudaStream_t st);
void launch_render(const DevCam* cams, const int* tile_view, int n_tiles, const int* tile_offsets,
                   const int* entries, const float4* rec, int Gp, const float* gt, float* image,
                   float* trans, int* contrib, int* last, double* sse_tile, cudaStream_t st,
                   unsigned long long* stats = nullptr);
void launch_render_exact(const DevCam* cams, const int* tile_view, int n_tiles, const int* tile_offsets,
                         const int* entries, const double* rec64, const float4* rec, int Gp, double* image,
                         double* trans, int* contrib, cudaStream_t st);
void launch_render_splats(int width, int height, int tiles_x, int n_tiles, const int* offsets, const int* list,
                          const double* splats, double* image, double* trans, int* contrib, cudaStream_t st);
void launch_render_pixel(int n, const double* splats, double px, double py, double* out, int* contrib,
                         cudaStream_t st);
void launch_sse_views(const DevCam* cams, int V, int n_tiles, const double* sse_tile, double* sse_view,
                      cudaStream_t st);
void launch_sample_raster(int mode, const SampleArgs& a, cudaStream_t st);
void launch_masks(const SampleArgs& a, cudaStream_t st);
void launch_alpha(const SampleArgs& a, cudaStream_t st);
void launch_mask_stats(const SampleArgs& a, unsigned long long* st, cudaStream_t stream);
void launch_diag_raster(const DiagArgs& a, cudaStream_t st);
void launch_tangents(const float* beta32, const float* p, int G, int Gp, const DevCam* cams, int V,
                     const float4* rec, float4* tan, const int* done, cudaStream_t st);
void launch_chain(const float* beta32, int G, int Gp, const DevCam* cams, int V, const float4* rec,
                  float* inter, const DetOrder& det, const float* p, float lambda, float* out, const int* done,
                  cudaStream_t st);
void launch_chain_range(const float* beta32, int G, int Gp, const DevCam* cams, int V, const float4* rec,
                        float* inter, const DetOrder& det, const float* p, float lambda, float* out,
                        const int* done, int g0, int g1, bool reduce, cudaStream_t st);
void launch_sum_ranks(void* const* srcs, int world, void* dst, size_t n, bool f64, cudaStream_t st);
void launch_diag_finalize(const float* beta32, int G, int Gp, const DevCam* cams, int V,
                          const float4* rec, float* diagacc, const DetOrder& det, float* out, cudaStream_t st);
void build_slot_order(const Group* groups, int n_groups, const int* gcount, const int* glist,
                      const long long* mask_off, const long long* wbase, int Gp, int V, long long n_slots,
                      unsigned* ka, unsigned* kb, unsigned* va, unsigned* vb, unsigned* hist, unsigned* part,
                      unsigned* perm, unsigned* seg, unsigned* dest, unsigned* fill, cudaStream_t st);
void launch_aos64_to_soa32(const double* aos, int G, int Gp, float* soa, cudaStream_t st);
void launch_aos64_to_soa32_range(const double* aos, int g0, int g1, int Gp, float* soa, cudaStream_t st);
void launch_soa32_to_aos64_range(const float* soa, int g0, int g1, int Gp, double* aos, cudaStream_t st);
void launch_tangents_range(const float* beta32, const float* p, int G, int Gp, const DevCam* cams, int V,
                           const float4* rec, float4* tan, const int* done, int g0, int g1, cudaStream_t st);
void launch_soa32_to_aos64(const float* soa, int G, int Gp, double* aos, cudaStream_t st);
void launch_set_to_beta(const double* m, const double* ls, const double* rot, const double* logit,
                        const double* col, int G, int Gp, double* beta, float* beta32, cudaStream_t st);
void launch_beta_to_set(const double* beta, int G, int Gp, double* m, double* ls, double* rot,
                        double* logit, double* col, cudaStream_t st);
void launch_dot(const float* a, const float* b, long long n, double* partial, double* out, cudaStream_t st);
void launch_color_maxabs(const float* x, int G, int Gp, float* out, cudaStream_t st);
void launch_cg_init(const float* b, const float* minv, long long n, float* x, float* r, float* z,
                    float* p, double* partial, CgState* s, cudaStream_t st);
void launch_cg_pu(const float* p, const float* u, long long n, double* partial, CgState* s, cudaStream_t st);
void launch_cg_update(float* x, float* r, float* z, float* p, const float* u, const float* minv,
                      long long n, double* partial, CgState* s, cudaStream_t st);
void launch_minv(float* d, long long n, float lambda, cudaStream_t st);
int metric_tiles(int w, int h, int* tiles_x);
void launch_image_metrics(const float* a, const float* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st);
void launch_image_metrics(const double* a, const double* b, const ImgDesc* imgs, int n_img, int max_tiles,
                          double2* partial, double2* out, const MetricWindow& win, cudaStream_t st);
void launch_ssim_diag(const float* a, const float* b, const ImgDesc* imgs, int n_img, int max_tiles,
                      double2* partial, double2* out, const MetricWindow& win, float* res, float* dcen,
                      cudaStream_t st);
void launch_ssim_diag(const double* a, const double* b, const ImgDesc* imgs, int n_img, int max_tiles,
                      double2* partial, double2* out, const MetricWindow& win, double* res, double* dcen,
                      cudaStream_t st);
void launch_ssim_fold(const Group* groups, int n_groups, const DevCam* cams, const int* spix, const int* sorig,
                      float* sw, const float* image, const float* gt, const float* sres, const float* sdc,
                      float ssim_weight, float* rhs, const float* scol, cudaStream_t st);
void launch_weighted_draw(const DevCam* cams, int n_tiles, const int* tile_view, const int* tile_sbase,
                          const double* image, const float* gt, const int* contrib, int dist, int spt,
                          const double* U, double n_total, double inv_total, int* spix, float* sw,
                          cudaStream_t st);
void launch_exhaustive_residual(const DevCam* cams, int n_tiles, const int* tile_view, const int* tile_sbase,
                                const float* image, const float* gt, const float* sres, const float* sdc,
                                float ssim_weight, float scale, int* spix, float* u, cudaStream_t st);
void launch_first_order_step(double* beta, float* beta32, double* m1, double* m2, const float* grad32,
                             const double* grad64_aos, int G, int Gp, const FirstOrderParams& fp, cudaStream_t st);
void launch_axpy(float* y, const float* x, long long n, float a, cudaStream_t st);
void launch_widen(const float* x, double* y, long long n, cudaStream_t st);
void launch_narrow(const double* x, float* y, long long n, cudaStream_t st);

}  // namespace slm
