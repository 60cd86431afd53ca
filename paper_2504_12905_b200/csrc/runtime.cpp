// runtime.cpp — host C++ runtime and C ABI of libslm_b200.so.
//
// Mirrors the reference's C++ solver API (proj/include/splatlm/**) on top of
// the sm_100a kernels: device-resident GaussianSet (Scene), the batch's
// prepared views and tile lists (Batch), the sample plan laid out as warp
// groups (Samples), SampledJacobian (Jacobian), the device PCG and lm_step.
// The samplers (build_sample_plan, k-means view batching, random_init) stay on
// the host with libstdc++'s <random>, which is what makes the sampled pixel
// sets bit-identical to the reference (SURVEY §7 hard part 2).
#include "runtime.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdlib>
#include <fstream>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>
#include <condition_variable>
#include <numeric>
#include <sstream>
#include <thread>

#include <dlfcn.h>
#include <nccl.h>

#include "slm_b200.h"

namespace slm {

std::atomic<long long> g_launches{0};

namespace {
thread_local std::string g_err;

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// NCCL is resolved at first use with dlopen, never at load time: the library
// must coexist with whichever libnccl.so.2 the host process (e.g. PyTorch's
// bundled 2.28) already mapped, and single-GPU use needs no NCCL at all.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    void* h = nullptr;
    if (const char* env = std::getenv("SLM_NCCL_LIB")) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw NcclError("NCCL library not found (set SLM_NCCL_LIB)");
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(dlsym(h, "ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy || !api.GetErrorString ||
        !api.GroupStart || !api.GroupEnd)
        throw NcclError("NCCL library lacks required symbols");
    loaded = true;
    return api;
}

#define SLM_NCCL_CHECK(x)                                                                  \
    do {                                                                                   \
        ncclResult_t r_ = (x);                                                             \
        if (r_ != ncclSuccess) throw NcclError(std::string("NCCL error: ") + nccl().GetErrorString(r_)); \
    } while (0)

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
}  // namespace

// =========================================================================== collectives
// The view-sharded path's collective seam: a sum-allreduce of f32 or
// f64 device vectors on the context's stream.  NcclComm: one process per GPU
// (the deployment).  LocalComm: a group of contexts inside ONE process -- on one
// GPU or several -- each rank driven by its own host thread; it sums the ranks'
// buffers in rank order (deterministic for a given world size), so the world > 1
// code path (view slices, [b | diag], products, loss scalars) runs and is tested
// on a single B200.
struct Comm {
    virtual ~Comm() = default;
    virtual void allreduce(void* p, size_t n, bool f64, cudaStream_t st) = 0;
    // f32 rows [base + r * pitch, + len), r < rows: one Gaussian chunk of a [14][Gp] vector
    virtual void allreduce_rows(float* base, size_t pitch, int rows, size_t len, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    ~NcclComm() override {
        if (c) nccl().CommDestroy(c);
    }
    void allreduce(void* p, size_t n, bool f64, cudaStream_t st) override {
        SLM_NCCL_CHECK(nccl().AllReduce(p, p, n, f64 ? ncclFloat64 : ncclFloat32, ncclSum, c, st));
    }
    void allreduce_rows(float* base, size_t pitch, int rows, size_t len, cudaStream_t st) override {
        SLM_NCCL_CHECK(nccl().GroupStart());
        for (int r = 0; r < rows; ++r)
            SLM_NCCL_CHECK(nccl().AllReduce(base + r * pitch, base + r * pitch, len, ncclFloat32, ncclSum, c, st));
        SLM_NCCL_CHECK(nccl().GroupEnd());
    }
};

// Host rendezvous + per-rank staging slots and events.  One allreduce round:
//   1. wait until every rank finished reading the staging slots of the last round
//   2. copy the rank's vector into its slot, record `ready`
//   3. barrier; wait for every rank's `ready`; sum the slots in rank order into
//      the rank's own vector (k_sum_ranks); record `done`; barrier.
struct LocalGroup {
    int world;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    std::vector<void*> slot;
    std::vector<size_t> slot_bytes;
    std::vector<int> slot_dev;
    std::vector<cudaEvent_t> ready, done;
    explicit LocalGroup(int w) : world(w), slot(w, nullptr), slot_bytes(w, 0), slot_dev(w, 0), ready(w, nullptr),
                                 done(w, nullptr) {}
    ~LocalGroup() {
        for (int r = 0; r < world; ++r) {
            if (slot[r]) cudaFree(slot[r]);
            if (ready[r]) cudaEventDestroy(ready[r]);
            if (done[r]) cudaEventDestroy(done[r]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const long long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

void launch_sum_ranks(void* const* srcs, int world, void* dst, size_t n, bool f64, cudaStream_t st);

struct LocalComm : Comm {
    std::shared_ptr<LocalGroup> g;
    int rank;
    int device;
    LocalComm(std::shared_ptr<LocalGroup> grp, int r, int dev) : g(std::move(grp)), rank(r), device(dev) {
        SLM_CUDA_CHECK(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
        SLM_CUDA_CHECK(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
        g->slot_dev[rank] = dev;
    }
    void allreduce(void* p, size_t n, bool f64, cudaStream_t st) override {
        const size_t bytes = n * (f64 ? 8 : 4);
        for (int k = 0; k < g->world; ++k)  // 1. the last round's readers are done with the slots
            SLM_CUDA_CHECK(cudaStreamWaitEvent(st, g->done[k], 0));
        if (g->slot_bytes[rank] < bytes) {  // grow this rank's slot (nobody reads it now)
            SLM_CUDA_CHECK(cudaStreamSynchronize(st));
            if (g->slot[rank]) SLM_CUDA_CHECK(cudaFree(g->slot[rank]));
            SLM_CUDA_CHECK(cudaMalloc(&g->slot[rank], bytes));
            g->slot_bytes[rank] = bytes;
        }
        SLM_CUDA_CHECK(cudaMemcpyAsync(g->slot[rank], p, bytes, cudaMemcpyDeviceToDevice, st));
        SLM_CUDA_CHECK(cudaEventRecord(g->ready[rank], st));
        g->barrier();
        for (int k = 0; k < g->world; ++k) {
            SLM_CUDA_CHECK(cudaStreamWaitEvent(st, g->ready[k], 0));
            if (g->slot_dev[k] != device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(g->slot_dev[k], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SLM_CUDA_CHECK(e);
                cudaGetLastError();
            }
        }
        launch_sum_ranks(g->slot.data(), g->world, p, n, f64, st);
        SLM_CUDA_CHECK(cudaEventRecord(g->done[rank], st));
        g->barrier();
    }
    float* rows_tmp = nullptr;
    size_t rows_cap = 0;
    ~LocalComm() override {
        if (rows_tmp) cudaFree(rows_tmp);
    }
    void allreduce_rows(float* base, size_t pitch, int rows, size_t len, cudaStream_t st) override {
        const size_t n = static_cast<size_t>(rows) * len;
        if (rows_cap < n) {
            SLM_CUDA_CHECK(cudaStreamSynchronize(st));
            if (rows_tmp) SLM_CUDA_CHECK(cudaFree(rows_tmp));
            SLM_CUDA_CHECK(cudaMalloc(&rows_tmp, n * sizeof(float)));
            rows_cap = n;
        }
        SLM_CUDA_CHECK(cudaMemcpy2DAsync(rows_tmp, len * sizeof(float), base, pitch * sizeof(float), len * sizeof(float),
                                         rows, cudaMemcpyDeviceToDevice, st));
        allreduce(rows_tmp, n, false, st);
        SLM_CUDA_CHECK(cudaMemcpy2DAsync(base, pitch * sizeof(float), rows_tmp, len * sizeof(float), len * sizeof(float),
                                         rows, cudaMemcpyDeviceToDevice, st));
    }
};

// =========================================================================== Context
struct StepBuffers;
void destroy_step(StepBuffers*);

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    cudaStream_t aux = nullptr;       // copy stream overlapping uploads with kernels on `stream`
    cudaEvent_t aux_done = nullptr;
    std::unique_ptr<Comm> comm;  // world > 1: NCCL (one process per GPU) or an in-process LocalGroup
    int rank = 0, world = 1;
    DevBuf<double> partial;
    DevBuf<CgState> cg;
    DevBuf<double> dscalar;
    DevBuf<float> fscalar;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    std::vector<double> last_timings;
    std::string last_timing_names;
    bool timing = false;
    bool prof = false;  // per-kernel CUDA events inside gn_apply_dev
    // J^T / diag accumulation in a fixed per-plan order (DetOrder) instead of
    // float red.global.add: bitwise run-to-run reproducible (the default)
    bool deterministic = true;
    std::vector<std::array<cudaEvent_t, 4>> prof_events;
    StepBuffers* step = nullptr;  // persistent lm_step workspace
    // counters of the last lm_step (for the bench's per-step algorithmic bytes):
    // [views, sum G_v, tile-list entries, samples, pixels, PCG iterations,
    //  sum G_v after the update, entries after the update]
    long long step_stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};

    explicit Context(int dev) : device(dev) {
        SLM_CUDA_CHECK(cudaSetDevice(dev));
        SLM_CUDA_CHECK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        partial.ensure(2 * kRedBlocks);
        cg.ensure(1);
        dscalar.ensure(16);
        fscalar.ensure(16);
    }
    ~Context() {
        destroy_step(step);
        for (auto& m : marks) cudaEventDestroy(m.second);
        comm.reset();
        if (stream && own_stream) cudaStreamDestroy(stream);
        if (aux) cudaStreamDestroy(aux);
        if (aux_done) cudaEventDestroy(aux_done);
        for (auto e : chunk_ev) cudaEventDestroy(e);
        if (comm_done) cudaEventDestroy(comm_done);
        if (comm_st) cudaStreamDestroy(comm_st);
    }
    // the chunked product allreduce: a comm stream and one event per chunk
    cudaStream_t comm_st = nullptr;
    std::vector<cudaEvent_t> chunk_ev;
    cudaEvent_t comm_done = nullptr;
    int comm_chunks = 4;
    cudaStream_t comm_stream() {
        if (!comm_st) {
            SLM_CUDA_CHECK(cudaStreamCreateWithFlags(&comm_st, cudaStreamNonBlocking));
            SLM_CUDA_CHECK(cudaEventCreateWithFlags(&comm_done, cudaEventDisableTiming));
        }
        return comm_st;
    }
    cudaEvent_t chunk_event(int i) {
        while (static_cast<int>(chunk_ev.size()) <= i) {
            cudaEvent_t e;
            SLM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            chunk_ev.push_back(e);
        }
        return chunk_ev[i];
    }
    cudaStream_t aux_stream() {
        if (!aux) {
            SLM_CUDA_CHECK(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking));
            SLM_CUDA_CHECK(cudaEventCreateWithFlags(&aux_done, cudaEventDisableTiming));
        }
        return aux;
    }
    void activate() const { SLM_CUDA_CHECK(cudaSetDevice(device)); }
    void sync() const { SLM_CUDA_CHECK(cudaStreamSynchronize(stream)); }
    void check_launch() const { SLM_CUDA_CHECK(cudaGetLastError()); }

    void mark(const char* name) {
        if (!timing) return;
        cudaEvent_t e;
        SLM_CUDA_CHECK(cudaEventCreate(&e));
        SLM_CUDA_CHECK(cudaEventRecord(e, stream));
        marks.emplace_back(name, e);
    }
    void finish_marks() {
        if (!timing || marks.empty()) return;
        sync();
        last_timings.clear();
        last_timing_names.clear();
        for (size_t i = 1; i < marks.size(); ++i) {
            last_timing_names += marks[i].first + (i + 1 < marks.size() ? "," : "");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            last_timings.push_back(ms);
        }
        for (auto& m : marks) cudaEventDestroy(m.second);
        marks.clear();
    }

    void prof_record(std::array<cudaEvent_t, 4>& ev, int i) {
        if (i == 0)
            for (auto& e : ev) SLM_CUDA_CHECK(cudaEventCreate(&e));
        SLM_CUDA_CHECK(cudaEventRecord(ev[i], stream));
    }
    // {tangents, raster, chain} summed ms and launch count since the last collect
    void prof_collect(double out[3], int* n) {
        sync();
        out[0] = out[1] = out[2] = 0.0;
        for (auto& ev : prof_events) {
            for (int k = 0; k < 3; ++k) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
                out[k] += ms;
            }
            for (auto& e : ev) cudaEventDestroy(e);
        }
        *n = static_cast<int>(prof_events.size());
        prof_events.clear();
    }

    void allreduce(float* p, size_t n) {
        if (world <= 1 || n == 0) return;
        comm->allreduce(p, n, false, stream);
    }
    void allreduce(double* p, size_t n) {
        if (world <= 1 || n == 0) return;
        comm->allreduce(p, n, true, stream);
    }
};

// =========================================================================== Scene
struct Scene {
    Context* ctx;
    int G = 0, Gp = 0;
    DevBuf<double> beta;    // f64 SoA [14][Gp]
    DevBuf<float> beta32;   // f32 mirror
    DevBuf<double> stage;   // host-layout staging (5 arrays)

    Scene(Context* c, const slm_gaussians& h) : ctx(c) { upload(h); }

    void upload(const slm_gaussians& h) {
        if (h.count < 0) throw std::invalid_argument("negative Gaussian count");
        ctx->activate();
        G = h.count;
        Gp = round_up(std::max(G, 1), 256);
        const size_t P = static_cast<size_t>(kP) * Gp;
        beta.ensure(P);
        beta32.ensure(P);
        SLM_CUDA_CHECK(cudaMemsetAsync(beta.p, 0, P * sizeof(double), ctx->stream));
        SLM_CUDA_CHECK(cudaMemsetAsync(beta32.p, 0, P * sizeof(float), ctx->stream));
        if (G == 0) return;
        stage.ensure(static_cast<size_t>(14) * G);
        double* s = stage.p;
        cudaStream_t st = ctx->stream;
        SLM_CUDA_CHECK(cudaMemcpyAsync(s, h.means, sizeof(double) * 3 * G, cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(s + 3 * G, h.log_scales, sizeof(double) * 3 * G, cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(s + 6 * G, h.rotations, sizeof(double) * 4 * G, cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(s + 10 * G, h.opacity_logits, sizeof(double) * G, cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(s + 11 * G, h.colors, sizeof(double) * 3 * G, cudaMemcpyHostToDevice, st));
        launch_set_to_beta(s, s + 3 * G, s + 6 * G, s + 10 * G, s + 11 * G, G, Gp, beta.p, beta32.p, st);
        ctx->check_launch();
    }

    void download(slm_gaussians& h) {
        if (h.count != G) throw std::invalid_argument("download: Gaussian count mismatch");
        if (G == 0) return;
        ctx->activate();
        stage.ensure(static_cast<size_t>(14) * G);
        double* s = stage.p;
        cudaStream_t st = ctx->stream;
        launch_beta_to_set(beta.p, G, Gp, s, s + 3 * G, s + 6 * G, s + 10 * G, s + 11 * G, st);
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.means, s, sizeof(double) * 3 * G, cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.log_scales, s + 3 * G, sizeof(double) * 3 * G, cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.rotations, s + 6 * G, sizeof(double) * 4 * G, cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.opacity_logits, s + 10 * G, sizeof(double) * G, cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.colors, s + 11 * G, sizeof(double) * 3 * G, cudaMemcpyDeviceToHost, st));
        ctx->sync();
    }

    size_t P() const { return static_cast<size_t>(kP) * Gp; }
};

// Page-locked host allocator: the per-step sample arrays are uploaded with
// cudaMemcpyAsync at DMA speed (grow-only vectors keep their capacity).
template <class T>
struct PinnedAlloc {
    using value_type = T;
    PinnedAlloc() = default;
    template <class U>
    PinnedAlloc(const PinnedAlloc<U>&) {}
    T* allocate(size_t n) {
        void* p = nullptr;
        if (cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocPortable) != cudaSuccess) throw std::bad_alloc();
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t) { cudaFreeHost(p); }
    template <class U>
    bool operator==(const PinnedAlloc<U>&) const { return true; }
    template <class U>
    bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
template <class T>
using pinned_vector = std::vector<T, PinnedAlloc<T>>;

// =========================================================================== Batch
// The prepared views of one scene state: splat records, tile lists (K1, K3,
// K4) and, after render(), the per-pixel forward state (K6).
struct Batch {
    Context* ctx;
    int V = 0, n_tiles = 0, Gp = 0, G = 0;
    long long n_pix = 0, n_entries = 0;
    std::vector<DevCam> hcams;
    std::vector<int> htile_view;
    pinned_vector<int> htile_offsets;  // CSR offsets of the tile lists (host copy, see wait_offsets)
    cudaEvent_t offs_ready = nullptr;
    DevBuf<DevCam> cams;
    DevBuf<int> tile_view, tile_offsets, entries, err;
    DevBuf<long long> total;
    DevBuf<float4> rec;
    DevBuf<double> rec64;  // FP64 [mx, my, a, b, c, o] per (view, Gaussian): exact blend decisions
    DevBuf<float4> conic;  // {A, B, C, opacity} per (view, Gaussian): the linearisation kernels' 16-B view
    DevBuf<unsigned long long> keys;
    DevBuf<short4> rect;
    DevBuf<float> image, trans, gt;
    DevBuf<int> contrib, last;
    DevBuf<double> sse_tile, sse_view;
    DevBuf<float> ssim_res, ssim_dc;  // mse+ssim loss: s and ds/dcentre per pixel and channel
    // FP64 replay of the reference's blend (k_render_exact): the mse+ssim loss
    // terms and SSIM planes and the weighted-distribution CDFs read it, so they
    // see the reference's render, not the FP32 one
    DevBuf<double> image64, trans64, gt64, ssim_res64, ssim_dc64;
    DevBuf<int> contrib64;
    bool rendered = false, has_gt = false, exact_rendered = false;
    std::vector<int> valid_count;  // G_v per view (counted by k_prepare)
    long long max_list = 0;        // longest tile list of the batch
    // radix tile-list construction scratch (sort.cu)
    DevBuf<unsigned long long> rk64a, rk64b, and_or, rruns;
    DevBuf<unsigned> rv32a, rv32b, rk32a, rk32b, rcount, rt32a, rt32b, rt32va, rt32vb, rhist, rpart;

    bool offsets_pending = false;
    explicit Batch(Context* c) : ctx(c) {}
    Batch(const Batch&) = delete;
    Batch& operator=(const Batch&) = delete;
    ~Batch() {
        if (offs_ready) cudaEventDestroy(offs_ready);
    }
    // htile_offsets / max_list are valid after this
    void wait_offsets() {
        if (!offsets_pending) return;
        SLM_CUDA_CHECK(cudaEventSynchronize(offs_ready));
        offsets_pending = false;
        max_list = 0;
        for (int t = 0; t < n_tiles; ++t)
            max_list = std::max<long long>(max_list, htile_offsets[t + 1] - htile_offsets[t]);
    }

    // geometry = false: a render-only batch (the LM step's loss_after) -- no FP64
    // geometry and no conic views (only the products and k_masks read them)
    void prepare(const Scene& s, const std::vector<slm_camera>& cv, bool geometry = true) {
        ctx->activate();
        cudaStream_t st = ctx->stream;
        V = static_cast<int>(cv.size());
        G = s.G;
        Gp = s.Gp;
        hcams.assign(V, DevCam{});
        htile_view.clear();
        n_tiles = 0;
        n_pix = 0;
        for (int v = 0; v < V; ++v) {
            const slm_camera& c = cv[v];
            if (c.width <= 0 || c.height <= 0) throw std::invalid_argument("camera size must be positive");
            if (c.width > 32767 * kTile || c.height > 32767 * kTile) throw std::invalid_argument("camera too large");
            DevCam& d = hcams[v];
            std::memcpy(d.R, c.world_to_cam, sizeof d.R);
            std::memcpy(d.t, c.translation, sizeof d.t);
            d.fx = c.fx;
            d.fy = c.fy;
            d.cx = c.cx;
            d.cy = c.cy;
            d.near_clip = c.near_clip;
            d.width = c.width;
            d.height = c.height;
            d.tiles_x = (c.width + kTile - 1) / kTile;
            d.tiles_y = (c.height + kTile - 1) / kTile;
            d.tile_base = n_tiles;
            d.pix_base = n_pix;
            n_tiles += d.tiles_x * d.tiles_y;
            n_pix += static_cast<long long>(c.width) * c.height;
            htile_view.insert(htile_view.end(), d.tiles_x * d.tiles_y, v);
        }
        cams.ensure(std::max(V, 1));
        tile_view.ensure(std::max(n_tiles, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(cams.p, hcams.data(), sizeof(DevCam) * V, cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(tile_view.p, htile_view.data(), sizeof(int) * n_tiles, cudaMemcpyHostToDevice, st));
        const size_t VG = static_cast<size_t>(V) * Gp;
        rec.ensure(3 * VG);
        rec64.ensure(6 * VG);
        conic.ensure(VG);
        keys.ensure(VG);
        rect.ensure(VG);
        tile_offsets.ensure(n_tiles + 1);
        total.ensure(2);
        err.ensure(1 + std::max(V, 1));
        SLM_CUDA_CHECK(cudaMemsetAsync(total.p, 0, sizeof(long long) * 2, st));
        SLM_CUDA_CHECK(cudaMemsetAsync(err.p, 0, sizeof(int) * (1 + V), st));
        // K1 + the entry total (sum of tile-rect areas); the per-tile offsets come
        // out of the sorted tile ids (build_tile_lists), so no per-tile atomics
        launch_prepare(s.beta.p, G, Gp, cams.p, V, rec.p, keys.p, rect.p,
                       reinterpret_cast<unsigned long long*>(total.p), err.p, geometry ? rec64.p : nullptr,
                       geometry ? conic.p : nullptr, st);
        // depth-sort keys in index order + the AND/OR of the valid keys (which
        // key bytes need a radix pass)
        const long long nvg = static_cast<long long>(V) * Gp;
        rk64a.ensure(std::max<long long>(nvg, 1));
        rk64b.ensure(std::max<long long>(nvg, 1));
        rv32a.ensure(std::max<long long>(nvg, 1));
        rv32b.ensure(std::max<long long>(nvg, 1));
        and_or.ensure(2);
        launch_depth_init(keys.p, rect.p, G, Gp, V, rk64a.p, rv32a.p, and_or.p, st);
        ctx->check_launch();
        ctx->mark("prep:project+count+scan");
        long long hdr[2];
        unsigned long long hao[2] = {0ull, 0ull};
        std::vector<int> herr(1 + V);
        SLM_CUDA_CHECK(cudaMemcpyAsync(hdr, total.p, 2 * sizeof(long long), cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(hao, and_or.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(herr.data(), err.p, sizeof(int) * (1 + V), cudaMemcpyDeviceToHost, st));
        ctx->sync();
        if (herr[0]) throw std::domain_error("zero-norm quaternion");
        valid_count.assign(herr.begin() + 1, herr.end());
        n_entries = hdr[0];
        if (n_entries >= (1ll << 31)) throw std::runtime_error("tile-list entries exceed 2^31");
        entries.ensure(std::max<long long>(n_entries, 1));
        ctx->mark("prep:sync");
        // tile lists by stable radix passes (sort.cu): depth ranks, emit, sort by tile
        const long long ne = std::max<long long>(n_entries, 1);
        rk32a.ensure(std::max<long long>(nvg, 1));
        rk32b.ensure(std::max<long long>(nvg, 1));
        rcount.ensure(std::max<long long>(nvg, 1));
        rt32a.ensure(ne);
        rt32b.ensure(ne);
        rt32va.ensure(ne);
        rt32vb.ensure(ne);
        const long long hmax = radix_hist_size(std::max<long long>(nvg, ne));
        rhist.ensure(hmax);
        rpart.ensure(scan_scratch(std::max<long long>(hmax, nvg)));
        rruns.ensure(1 + 2 * (nvg / 33 + 1));
        TileSortBuffers tb{rk64a.p, rk64b.p, rv32a.p, rv32b.p, rk32a.p, rk32b.p, rcount.p,
                           rt32a.p, rt32b.p, rt32va.p, rt32vb.p, rhist.p, rpart.p, rruns.p};
        build_tile_lists(keys.p, rect.p, cams.p, G, Gp, V, n_tiles, n_entries, hao[0], hao[1], tb, entries.p,
                         tile_offsets.p, st);
        ctx->check_launch();
        // host copy of the offsets (Samples::upload needs them): async into pinned
        // memory, waited for only where it is read (wait_offsets)
        htile_offsets.resize(n_tiles + 1);
        SLM_CUDA_CHECK(cudaMemcpyAsync(htile_offsets.data(), tile_offsets.p, sizeof(int) * (n_tiles + 1),
                                       cudaMemcpyDeviceToHost, st));
        if (!offs_ready) SLM_CUDA_CHECK(cudaEventCreateWithFlags(&offs_ready, cudaEventDisableTiming));
        SLM_CUDA_CHECK(cudaEventRecord(offs_ready, st));
        offsets_pending = true;
        ctx->mark("prep:sort");
        rendered = false;
        has_gt = false;
        exact_rendered = false;
    }

    // render_full (rasterizer.cpp:93-95) of every pixel in FP64 (k_render_exact)
    void render_exact() {
        if (exact_rendered) return;
        image64.ensure(3 * std::max<long long>(n_pix, 1));
        trans64.ensure(std::max<long long>(n_pix, 1));
        contrib64.ensure(std::max<long long>(n_pix, 1));
        launch_render_exact(cams.p, tile_view.p, n_tiles, tile_offsets.p, entries.p, rec64.p, rec.p, Gp, image64.p,
                            trans64.p, contrib64.p, ctx->stream);
        ctx->check_launch();
        ctx->mark("render_exact");
        exact_rendered = true;
    }
    // the truth images widened to f64 (after copy_gt)
    void widen_gt() {
        gt64.ensure(3 * std::max<long long>(n_pix, 1));
        launch_widen(gt.p, gt64.p, 3 * n_pix, ctx->stream);
    }

    // Forward render of every pixel of every view (K6); gt (concatenated f32
    // H*W*3 per view, device) enables the per-view SSE.
    // full: also T, contrib and `last` per pixel (the drop-in render); the
    // LM step's loss renders and the metrics need only colour (+ SSE).
    void render(bool with_gt, bool full = true) {
        cudaStream_t st = ctx->stream;
        image.ensure(3 * std::max<long long>(n_pix, 1));
        if (full) {
            trans.ensure(std::max<long long>(n_pix, 1));
            contrib.ensure(std::max<long long>(n_pix, 1));
            last.ensure(std::max<long long>(n_pix, 1));
        }
        sse_tile.ensure(std::max(n_tiles, 1));
        sse_view.ensure(std::max(V, 1));
        launch_render(cams.p, tile_view.p, n_tiles, tile_offsets.p, entries.p, rec.p, Gp,
                      with_gt ? gt.p : nullptr, image.p, full ? trans.p : nullptr, full ? contrib.p : nullptr,
                      full ? last.p : nullptr, with_gt ? sse_tile.p : nullptr, st);
        if (with_gt) launch_sse_views(cams.p, V, n_tiles, sse_tile.p, sse_view.p, st);
        ctx->check_launch();
        ctx->mark("render");
        rendered = true;
        has_gt = with_gt;
    }

    std::vector<double> view_sse() {
        std::vector<double> h(V);
        if (V == 0) return h;
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.data(), sse_view.p, sizeof(double) * V, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        return h;
    }
};


// =========================================================================== Samples
// A plan laid out for the warp-per-group raster: per view, samples grouped
// by tile in chunks of <= 32 (the reference emits them tile-major already,
// sample_plan.cpp:96-168, so this is a no-op permutation for its plans).
struct Samples {
    pinned_vector<Group> hgroups;
    DevBuf<Group> groups;
    DevBuf<int> spix, sorig;
    DevBuf<float> sw, scol;  // scol: per-sample C_final of the FP64 blend (k_masks)
    DevBuf<long long> mask_off;
    DevBuf<unsigned> masks, cols;
    DevBuf<int> glist, gcount, grows;
    DevBuf<long long> srow_off, wbase;
    DevBuf<float> astream, rstream;
    // deterministic accumulation (DetOrder): slot sort scratch, order, partials
    DevBuf<unsigned> dka, dkb, dva, dvb, dhist, dpart, perm, seg, dest, fill;
    DevBuf<float> partial;
    long long n_slots = 0;
    std::vector<int> hrows, hcount;
    std::vector<long long> hrow_off, hwbase;
    std::vector<int> order;  // group order -> plan sample index
    pinned_vector<int> hpix, horig;
    pinned_vector<float> hw;
    long long total = 0, mask_words = 0;
    bool device_drawn = false;  // spix / sw written on the device (weighted distributions)

    // Host half (no CUDA calls; runs on the sampler thread in lm_step):
    // group the plan's samples per view by tile in chunks of <= 32, and the
    // per-sample f32 weights (1/q)/N_total (jacobian.cpp:112-116) for the raster.
    // w1 (optional) receives the f64 weight per sample.  One pass for the
    // reference's tile-major plans; other orders are stably sorted by tile.
    void group_host(const slm_plan& plan, int view_lo, int view_hi, const std::vector<slm_camera>& cams,
                    double inv_total, std::vector<double>* w1) {
        device_drawn = false;
        hgroups.clear();
        order.clear();
        const long long a0 = plan.view_offset[view_lo], n_all = plan.view_offset[view_hi] - a0;
        hpix.resize(n_all);
        horig.resize(n_all);
        hw.resize(3 * n_all);
        if (w1) w1->resize(n_all);
        long long k = 0;  // group-order position
        std::vector<int> idx;
        for (int v = view_lo; v < view_hi; ++v) {
            const slm_camera& c = cams[v - view_lo];
            const int tiles = ((c.width + kTile - 1) / kTile) * ((c.height + kTile - 1) / kTile);
            const long long a = plan.view_offset[v], b = plan.view_offset[v + 1];
            bool sorted = true;
            for (long long s = a; s < b; ++s) {
                if (plan.px[s] < 0 || plan.px[s] >= c.width || plan.py[s] < 0 || plan.py[s] >= c.height)
                    throw std::invalid_argument("sample pixel outside the camera");
                if (plan.tile[s] < 0 || plan.tile[s] >= tiles)
                    throw std::invalid_argument("sample tile outside the camera");
                if (s > a && plan.tile[s] < plan.tile[s - 1]) sorted = false;
            }
            const int* ord = nullptr;  // plan index of the view's i-th sample in tile order
            if (!sorted) {
                idx.resize(b - a);
                std::iota(idx.begin(), idx.end(), static_cast<int>(a));
                std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return plan.tile[x] < plan.tile[y]; });
                ord = idx.data();
            }
            long long i = 0;
            const long long n = b - a;
            while (i < n) {
                const long long s0 = ord ? ord[i] : a + i;
                const int t = plan.tile[s0];
                long long j = i;
                while (j < n && plan.tile[ord ? ord[j] : a + j] == t && j - i < 32) ++j;
                hgroups.push_back(Group{v - view_lo, t, static_cast<int>(k), static_cast<int>(j - i)});
                for (long long q = i; q < j; ++q, ++k) {
                    const long long s = ord ? ord[q] : a + q;
                    if (ord) order.push_back(static_cast<int>(s));
                    hpix[k] = plan.px[s] | (plan.py[s] << 16);
                    horig[k] = static_cast<int>(s - a0);
                    const double w = plan.weight[s] * inv_total;
                    if (w1) (*w1)[s - a0] = w;
                    const float wf = static_cast<float>(w);
                    hw[3 * k] = wf;
                    hw[3 * k + 1] = wf;
                    hw[3 * k + 2] = wf;
                }
                i = j;
            }
        }
        total = k;
        if (order.empty()) {  // identity (tile-major plans): spelled out for take_host / upload users
            order.resize(total);
            std::iota(order.begin(), order.end(), static_cast<int>(a0));
        }
    }

    // Host half of a device-drawn plan (weighted distributions): min(N, m)
    // draws per tile in plan order (tile-major), grouped in chunks of <= 32;
    // the pixels and weights are filled in by k_weighted_draw.  Returns the
    // first sample of every tile (batch tile order).
    std::vector<int> group_tiles_host(const std::vector<slm_camera>& cams, int spt) {
        device_drawn = true;
        hgroups.clear();
        order.clear();
        std::vector<int> sbase;
        for (int v = 0; v < static_cast<int>(cams.size()); ++v) {
            const slm_camera& c = cams[v];
            const int txn = (c.width + kTile - 1) / kTile, tyn = (c.height + kTile - 1) / kTile;
            for (int t = 0; t < txn * tyn; ++t) {
                const int w = std::min(c.width - (t % txn) * kTile, kTile);
                const int h = std::min(c.height - (t / txn) * kTile, kTile);
                const int n = std::min(spt, w * h);
                sbase.push_back(static_cast<int>(order.size()));
                for (int i = 0; i < n; i += 32) {
                    const int cnt = std::min(32, n - i);
                    hgroups.push_back(Group{v, t, static_cast<int>(order.size()), cnt});
                    for (int k = 0; k < cnt; ++k) order.push_back(static_cast<int>(order.size()));
                }
            }
        }
        total = static_cast<long long>(order.size());
        horig.resize(order.size());
        for (size_t k = 0; k < order.size(); ++k) horig[k] = static_cast<int>(k);
        hpix.assign(order.size(), 0);
        hw.assign(3 * order.size(), 0.f);
        return sbase;
    }

    // Device half: mask offsets (need the tile-list lengths) and uploads.
    pinned_vector<long long> hoff;
    void upload(Context* ctx, const std::vector<DevCam>& cams, const pinned_vector<int>& tile_offsets,
                cudaStream_t st) {
        hoff.resize(hgroups.size());
        mask_words = 0;
        for (size_t g = 0; g < hgroups.size(); ++g) {
            const int t = cams[hgroups[g].view].tile_base + hgroups[g].tile;
            const long long n = tile_offsets[t + 1] - tile_offsets[t];
            hoff[g] = mask_words;
            mask_words += 32 * ((n + 31) / 32);
        }
        (void)ctx;
        mask_off.ensure(std::max<size_t>(hoff.size(), 1));
        masks.ensure(std::max<long long>(mask_words, 1));
        cols.ensure(std::max<long long>(mask_words, 1));
        glist.ensure(std::max<long long>(mask_words, 1));
        gcount.ensure(std::max<size_t>(hgroups.size(), 1));
        grows.ensure(std::max<size_t>(hgroups.size(), 1));
        srow_off.ensure(std::max<size_t>(hgroups.size(), 1));
        wbase.ensure(std::max<size_t>(hgroups.size(), 1));
        groups.ensure(std::max<size_t>(hgroups.size(), 1));
        spix.ensure(std::max<size_t>(order.size(), 1));
        sorig.ensure(std::max<size_t>(order.size(), 1));
        sw.ensure(std::max<size_t>(3 * order.size(), 1));
        scol.ensure(std::max<size_t>(3 * order.size(), 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(mask_off.p, hoff.data(), sizeof(long long) * hoff.size(), cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(groups.p, hgroups.data(), sizeof(Group) * hgroups.size(), cudaMemcpyHostToDevice, st));
        SLM_CUDA_CHECK(cudaMemcpyAsync(sorig.p, horig.data(), sizeof(int) * horig.size(), cudaMemcpyHostToDevice, st));
        if (!device_drawn) {
            SLM_CUDA_CHECK(cudaMemcpyAsync(spix.p, hpix.data(), sizeof(int) * hpix.size(), cudaMemcpyHostToDevice, st));
            SLM_CUDA_CHECK(cudaMemcpyAsync(sw.p, hw.data(), sizeof(float) * hw.size(), cudaMemcpyHostToDevice, st));
        }
        // (host arrays are pinned members, rewritten only after later syncs)
    }

    void upload_weights(Context* ctx, const std::vector<double>& weights3) {
        for (size_t k = 0; k < order.size(); ++k)
            for (int c = 0; c < 3; ++c) hw[3 * k + c] = static_cast<float>(weights3[3 * static_cast<size_t>(horig[k]) + c]);
        SLM_CUDA_CHECK(cudaMemcpyAsync(sw.p, hw.data(), sizeof(float) * hw.size(), cudaMemcpyHostToDevice, ctx->stream));
        ctx->sync();
    }
};

// =========================================================================== Jacobian
struct Jacobian {
    Context* ctx;
    Scene* scene;                    // parameters (owned or borrowed)
    std::unique_ptr<Scene> own_scene;
    Batch* batch;
    std::unique_ptr<Batch> own_batch;
    Samples samples;
    std::vector<double> weights;     // (1/q)/N_total per residual, (view, sample, channel)
    long long rdim = 0, plan_base = 0;
    DevBuf<float4> tan;
    DevBuf<float> inter, diagacc, vin, vout, res_in, res_out;
    DevBuf<double> host_stage;
    DevBuf<float> r, z, p, u;

    Jacobian(Context* c, Scene* s, Batch* b) : ctx(c), scene(s), batch(b) {}

    // plan views [lo, hi) are this rank's; the weights use the global N_total.
    // Host half: residual weights (jacobian.cpp:112-116) and sample grouping.
    // Pure host work, safe to run concurrently with GPU work on the context.
    void init_host(const slm_plan& plan, int lo, int hi, double inv_total, const std::vector<slm_camera>& cams) {
        draw.on = false;
        draw.exhaustive = false;
        rdim = 0;
        plan_base = plan.view_offset[lo];
        for (int v = lo; v < hi; ++v) rdim += 3 * (plan.view_offset[v + 1] - plan.view_offset[v]);
        weights.clear();  // materialised on demand (residual_weights): lm_step never reads them
        samples.group_host(plan, lo, hi, cams, inv_total, &w1);
    }
    std::vector<double> w1;  // (1/q)/N_total per sample (plan order), all three channels
    const std::vector<double>& residual_weights() {
        if (weights.empty() && !w1.empty() && static_cast<long long>(w1.size()) * 3 == rdim) {
            weights.resize(rdim);
            for (size_t k = 0; k < w1.size(); ++k)
                for (int c = 0; c < 3; ++c) weights[3 * k + c] = w1[k];
        }
        return weights;
    }

    // Weighted residual distributions (sample_plan.cpp:127-165): the host draws
    // the uniforms from the caller's RNG in the reference's order, the device
    // picks the pixels from the per-tile CDFs of the render (sampler.cu).
    struct Draw {
        bool on = false;
        bool exhaustive = false;  // full_gradient: every pixel + u = 2/M (r + w s s') (first_order.cu)
        const float* sres = nullptr;
        const float* sdc = nullptr;
        float ssim_weight = 0.f, scale = 0.f;
        int dist = 0, spt = 0;
        double n_total = 0.0, inv_total = 0.0;
        pinned_vector<double> hU;
        std::vector<int> hsbase;
        DevBuf<double> U;
        DevBuf<int> sbase;
    } draw;

    void init_host_weighted(const std::vector<slm_camera>& all, int lo, int hi, int spt, int dist, int lane,
                            std::mt19937_64& rng) {
        if (spt < 1) throw std::invalid_argument("samples_per_tile must be positive");
        if (spt > kTile * kTile) throw std::invalid_argument("samples_per_tile exceeds the pixels in a tile");
        if (lane < 1 || spt % lane != 0)
            throw std::invalid_argument("samples_per_tile must be a multiple of the lane width");
        if (dist != SLM_DIST_RESIDUAL && dist != SLM_DIST_GAUSSIAN_COUNT)
            throw std::invalid_argument("unknown residual distribution");
        long long total = 0, off_lo = 0, off_hi = 0;
        for (int v = 0; v < static_cast<int>(all.size()); ++v) {
            if (v == lo) off_lo = total;
            const int txn = (all[v].width + kTile - 1) / kTile, tyn = (all[v].height + kTile - 1) / kTile;
            for (int ty = 0; ty < tyn; ++ty)
                for (int tx = 0; tx < txn; ++tx)
                    total += std::min(spt, std::min(all[v].width - tx * kTile, kTile) *
                                               std::min(all[v].height - ty * kTile, kTile));
            if (v + 1 == hi) off_hi = total;
        }
        if (lo >= hi) off_lo = off_hi = 0;
        // one uniform per draw, every rank replays the whole batch (draw_from_cdf, :53-58)
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        draw.hU.resize(std::max<long long>(off_hi - off_lo, 1));
        for (long long i = 0; i < total; ++i) {
            const double u = uni(rng);
            if (i >= off_lo && i < off_hi) draw.hU[i - off_lo] = u;
        }
        draw.on = true;
        draw.exhaustive = false;
        draw.dist = dist;
        draw.spt = spt;
        draw.n_total = static_cast<double>(total);
        draw.inv_total = total > 0 ? 1.0 / static_cast<double>(total) : 0.0;
        const std::vector<slm_camera> mine(all.begin() + lo, all.begin() + hi);
        draw.hsbase = samples.group_tiles_host(mine, spt);
        rdim = 3 * samples.total;
        plan_base = off_lo;
        weights.clear();  // drawn on the device (lm_step's Jacobian never reads them on the host)
        w1.clear();
    }

    // Host half of full_gradient's exhaustive plan (sample_plan.cpp:173-197)
    // over these cameras, laid out tile-major for the raster; u is filled on
    // the device (first_order.cu) in the same order.
    void init_host_exhaustive(const std::vector<slm_camera>& cams, const float* sres, const float* sdc,
                              float ssim_weight, float scale) {
        draw.hsbase = samples.group_tiles_host(cams, kTile * kTile);
        draw.on = true;
        draw.exhaustive = true;
        draw.sres = sres;
        draw.sdc = sdc;
        draw.ssim_weight = ssim_weight;
        draw.scale = scale;
        rdim = 3 * samples.total;
        plan_base = 0;
        weights.clear();
        w1.clear();
    }

    // Adopt the host half computed by another (host-only) Jacobian.
    void take_host(Jacobian& o) {
        std::swap(draw.on, o.draw.on);
        std::swap(draw.exhaustive, o.draw.exhaustive);
        std::swap(draw.dist, o.draw.dist);
        std::swap(draw.spt, o.draw.spt);
        std::swap(draw.n_total, o.draw.n_total);
        std::swap(draw.inv_total, o.draw.inv_total);
        draw.hU.swap(o.draw.hU);
        draw.hsbase.swap(o.draw.hsbase);
        std::swap(samples.device_drawn, o.samples.device_drawn);
        std::swap(rdim, o.rdim);
        std::swap(plan_base, o.plan_base);
        weights.swap(o.weights);
        w1.swap(o.w1);
        samples.hgroups.swap(o.samples.hgroups);
        samples.order.swap(o.samples.order);
        samples.hpix.swap(o.samples.hpix);
        samples.horig.swap(o.samples.horig);
        samples.hw.swap(o.samples.hw);
        std::swap(samples.total, o.samples.total);
    }

    // Device half: uploads, zeroed accumulators, blend masks (needs the batch
    // prepared and rendered).
    // The plan's H2D uploads on the context's copy stream, so they overlap
    // whatever runs on the main stream (lm_step: the render); init_device waits.
    bool preuploaded = false;
    void upload_early() {
        cudaStream_t a = ctx->aux_stream();
        batch->wait_offsets();
        samples.upload(ctx, batch->hcams, batch->htile_offsets, a);
        SLM_CUDA_CHECK(cudaEventRecord(ctx->aux_done, a));
        preuploaded = true;
    }

    void init_device() {
        if (preuploaded) {
            SLM_CUDA_CHECK(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
            preuploaded = false;
        } else {
            batch->wait_offsets();
            samples.upload(ctx, batch->hcams, batch->htile_offsets, ctx->stream);
        }
        if (draw.on && draw.exhaustive) {  // exhaustive plan: pixels + dL/dr in sample order
            draw.sbase.ensure(std::max<size_t>(draw.hsbase.size(), 1));
            res_in.ensure(std::max<long long>(rdim, 1));
            SLM_CUDA_CHECK(cudaMemcpyAsync(draw.sbase.p, draw.hsbase.data(), sizeof(int) * draw.hsbase.size(),
                                           cudaMemcpyHostToDevice, ctx->stream));
            launch_exhaustive_residual(batch->cams.p, batch->n_tiles, batch->tile_view.p, draw.sbase.p,
                                       batch->image.p, batch->gt.p, draw.sres, draw.sdc, draw.ssim_weight,
                                       draw.scale, samples.spix.p, res_in.p, ctx->stream);
            ctx->check_launch();
        } else if (draw.on) {  // weighted distributions: pixels + weights from the render's CDFs
            draw.U.ensure(draw.hU.size());
            draw.sbase.ensure(std::max<size_t>(draw.hsbase.size(), 1));
            SLM_CUDA_CHECK(cudaMemcpyAsync(draw.U.p, draw.hU.data(), sizeof(double) * draw.hU.size(),
                                           cudaMemcpyHostToDevice, ctx->stream));
            SLM_CUDA_CHECK(cudaMemcpyAsync(draw.sbase.p, draw.hsbase.data(), sizeof(int) * draw.hsbase.size(),
                                           cudaMemcpyHostToDevice, ctx->stream));
            batch->render_exact();  // the reference's CDFs come from its f64 render_full (sample_plan.cpp:127-165)
            launch_weighted_draw(batch->cams.p, batch->n_tiles, batch->tile_view.p, draw.sbase.p, batch->image64.p,
                                 batch->gt.p, batch->contrib64.p, draw.dist, draw.spt, draw.U.p, draw.n_total,
                                 draw.inv_total, samples.spix.p, samples.sw.p, ctx->stream);
            ctx->check_launch();
        }
        ctx->mark("plan:upload");
        const size_t VG = static_cast<size_t>(batch->V) * scene->Gp;
        tan.ensure(3 * VG);
        det = ctx->deterministic;
        if (!det) {  // red.global.add accumulators (k_chain / k_diag_finalize re-zero them)
            inter.ensure(VG * kRec);
            diagacc.ensure(VG * kDiagRec);
            SLM_CUDA_CHECK(cudaMemsetAsync(inter.p, 0, VG * kRec * sizeof(float), ctx->stream));
            SLM_CUDA_CHECK(cudaMemsetAsync(diagacc.p, 0, VG * kDiagRec * sizeof(float), ctx->stream));
        }
        SLM_CUDA_CHECK(cudaMemsetAsync(tan.p, 0, 3 * VG * sizeof(float4), ctx->stream));
        // the blend masks depend on the state only: computed once per (state, plan)
        SampleArgs a = args();
        a.scol_out = samples.scol.p;
        a.masks_out = samples.masks.p;
        a.glist_out = samples.glist.p;
        a.gcount_out = samples.gcount.p;
        a.grows_out = samples.grows.p;
        launch_masks(a, ctx->stream);
        ctx->check_launch();
        ctx->mark("plan:masks");
        // alpha-stream layout: rows per group -> offsets (host scan), then the stream
        const size_t ng = samples.hgroups.size();
        samples.hrows.resize(ng);
        samples.hcount.resize(ng);
        samples.hrow_off.resize(ng);
        samples.hwbase.resize(ng);
        if (ng) {
            SLM_CUDA_CHECK(cudaMemcpyAsync(samples.hrows.data(), samples.grows.p, sizeof(int) * ng,
                                           cudaMemcpyDeviceToHost, ctx->stream));
            SLM_CUDA_CHECK(cudaMemcpyAsync(samples.hcount.data(), samples.gcount.p, sizeof(int) * ng,
                                           cudaMemcpyDeviceToHost, ctx->stream));
        }
        ctx->sync();
        long long rows = 0, wins = 0;
        for (size_t g = 0; g < ng; ++g) {
            samples.hrow_off[g] = rows;
            rows += samples.hrows[g];
            samples.hwbase[g] = wins;
            wins += (samples.hcount[g] + 31) / 32;
        }
        samples.astream.ensure(std::max<long long>(32 * rows, 1));
        samples.rstream.ensure(std::max<long long>(static_cast<long long>(kRecBlock) * wins, 1));
        if (ng) {
            SLM_CUDA_CHECK(cudaMemcpyAsync(samples.srow_off.p, samples.hrow_off.data(), sizeof(long long) * ng,
                                           cudaMemcpyHostToDevice, ctx->stream));
            SLM_CUDA_CHECK(cudaMemcpyAsync(samples.wbase.p, samples.hwbase.data(), sizeof(long long) * ng,
                                           cudaMemcpyHostToDevice, ctx->stream));
        }
        ctx->mark("plan:rows");
        SampleArgs b = args();
        b.astream_out = samples.astream.p;
        b.rstream_out = samples.rstream.p;
        b.cols_out = samples.cols.p;
        launch_alpha(b, ctx->stream);
        ctx->check_launch();
        ctx->mark("plan:alpha");
        if (det) {  // the fixed summation order of this plan's J^T / diag slots
            const long long ns = 32 * wins;
            samples.n_slots = ns;
            const long long nk = static_cast<long long>(batch->V) * scene->Gp;
            const long long n1 = std::max<long long>(ns, 1);
            samples.dka.ensure(n1);
            samples.dkb.ensure(n1);
            samples.dva.ensure(n1);
            samples.dvb.ensure(n1);
            samples.perm.ensure(n1);
            samples.dest.ensure(n1);
            samples.seg.ensure(nk + 1);
            // slot order: counting placement + per-key segment sort when keys carry a
            // few slots each (the segment sort is serial per key), else the stable
            // radix passes (SLM_SLOT_ORDER=radix|counting overrides)
            const char* so = std::getenv("SLM_SLOT_ORDER");
            const bool counting = so ? std::strcmp(so, "radix") != 0 : ns <= 4 * static_cast<long long>(batch->V) * scene->G;
            if (counting) samples.fill.ensure(nk);
            const long long hs = radix_hist_size(n1);
            samples.dhist.ensure(hs);
            samples.dpart.ensure(scan_scratch(std::max<long long>(hs, nk)));
            samples.partial.ensure(static_cast<size_t>(kDetDiagRec) * n1);  // J^T and diag records share it
            // summation path (DetOrder::fused): the chain thread sums its own keys when
            // keys carry few records each, else a record-parallel segmented reduction
            // first (few Gaussians, many records per key; SLM_DET_PATH=fused|reduce overrides)
            const char* env = std::getenv("SLM_DET_PATH");
            det_fused = env ? std::strcmp(env, "reduce") != 0 : ns <= 4 * static_cast<long long>(batch->V) * scene->G;
            if (!det_fused) {
                inter.ensure(static_cast<size_t>(nk) * kRec);
                diagacc.ensure(static_cast<size_t>(nk) * kDiagRec);
            }
            build_slot_order(samples.groups.p, static_cast<int>(ng), samples.gcount.p, samples.glist.p,
                             samples.mask_off.p, samples.wbase.p, scene->Gp, batch->V, ns, samples.dka.p,
                             samples.dkb.p, samples.dva.p, samples.dvb.p, samples.dhist.p, samples.dpart.p,
                             samples.perm.p, samples.seg.p, samples.dest.p, counting ? samples.fill.p : nullptr,
                             ctx->stream);
            ctx->check_launch();
        }
        ctx->sync();  // hrow_off is read by the async copy
    }

    bool det = true;  // this plan's accumulation mode (Context::deterministic at init_device)
    bool det_fused = true;
    DetOrder det_order() const {
        return det ? DetOrder{samples.seg.p, samples.partial.p, det_fused ? 1 : 0} : DetOrder{nullptr, nullptr, 0};
    }
    // out = sum_v chain_v^T inter_v (+ lambda p): the J^T chain of the last J^T pass
    void chain(const float* p, float lambda, float* out, const int* done = nullptr) {
        launch_chain(scene->beta32.p, scene->G, scene->Gp, batch->cams.p, batch->V, batch->conic.p, inter.p,
                     det_order(), p, lambda, out, done, ctx->stream);
    }

    SampleArgs args() const {
        SampleArgs a{};
        a.groups = samples.groups.p;
        a.n_groups = static_cast<int>(samples.hgroups.size());
        a.cams = batch->cams.p;
        a.tile_offsets = batch->tile_offsets.p;
        a.entries = batch->entries.p;
        a.rec = batch->rec.p;
        a.tan = tan.p;
        a.Gp = scene->Gp;
        a.spix = samples.spix.p;
        a.sorig = samples.sorig.p;
        a.sw = samples.sw.p;
        a.image = batch->image.p;
        a.last_img = batch->last.p;
        a.gt = batch->gt.p;
        a.inter = inter.p;
        a.partial = det ? samples.partial.p : nullptr;
        a.dest = samples.dest.p;
        a.masks = samples.masks.p;
        a.glist = samples.glist.p;
        a.gcount = samples.gcount.p;
        a.mask_off = samples.mask_off.p;
        a.srow_off = samples.srow_off.p;
        a.astream = samples.astream.p;
        a.wbase = samples.wbase.p;
        a.rstream = samples.rstream.p;
        a.cols = samples.cols.p;
        a.rec64 = batch->rec64.p;
        a.scol = samples.scol.p;
        return a;
    }

    size_t P() const { return scene->P(); }

    // out = J^T W J p + lambda p, device f32 SoA; allreduced across ranks.
    void gn_apply_dev(float lambda, const float* dp, float* dout, const int* done = nullptr) {
        cudaStream_t st = ctx->stream;
        std::array<cudaEvent_t, 4> ev{};
        const bool prof = ctx->prof;
        if (prof) ctx->prof_record(ev, 0);
        launch_tangents(scene->beta32.p, dp, scene->G, scene->Gp, batch->cams.p, batch->V, batch->conic.p,
                        tan.p, done, st);
        if (prof) ctx->prof_record(ev, 1);
        SampleArgs a = args();
        a.done_flag = done;
        launch_sample_raster(kGn, a, st);
        if (prof) ctx->prof_record(ev, 2);
        if (ctx->world > 1) {
            // chunk-pipelined chain + allreduce: the chain runs over
            // Gaussian chunks on the main stream; each finished chunk's 14 rows are
            // allreduced on the comm stream while the next chunk computes.  Rank 0
            // adds lambda p inside its chain, so the sum carries it exactly once.
            cudaStream_t cs = ctx->comm_stream();
            const int G = scene->G, Gp = scene->Gp;
            const int nch = std::max(1, ctx->comm_chunks);
            const int step = round_up((G + nch - 1) / nch, 256);
            const float* pp = ctx->rank == 0 ? dp : nullptr;
            int c = 0;
            for (int g0 = 0; g0 < G; g0 += step, ++c) {
                const int g1 = std::min(G, g0 + step);
                launch_chain_range(scene->beta32.p, G, Gp, batch->cams.p, batch->V, batch->conic.p, inter.p,
                                   det_order(), pp, lambda, dout, done, g0, g1, c == 0, st);
                SLM_CUDA_CHECK(cudaEventRecord(ctx->chunk_event(c), st));
                SLM_CUDA_CHECK(cudaStreamWaitEvent(cs, ctx->chunk_event(c), 0));
                ctx->comm->allreduce_rows(dout + g0, static_cast<size_t>(Gp), kP, static_cast<size_t>(g1 - g0), cs);
            }
            SLM_CUDA_CHECK(cudaEventRecord(ctx->comm_done, cs));
            SLM_CUDA_CHECK(cudaStreamWaitEvent(st, ctx->comm_done, 0));
        } else {
            chain(dp, lambda, dout, done);
        }
        if (prof) {
            ctx->prof_record(ev, 3);
            ctx->prof_events.push_back(ev);
        }
        ctx->check_launch();
    }

    // mse+ssim (lm.cpp:86-121): u = -w (r + ssim_weight sp sv) at the samples
    // from the batch's SSIM planes, then w <- w (1 + ssim_weight sp^2) for the
    // diag and the products; b = J^T u.
    void rhs_ssim_dev(float* dout, float ssim_weight) {
        res_in.ensure(std::max<long long>(rdim, 1));
        launch_ssim_fold(samples.groups.p, static_cast<int>(samples.hgroups.size()), batch->cams.p, samples.spix.p,
                         samples.sorig.p, samples.sw.p, batch->image.p, batch->gt.p, batch->ssim_res.p,
                         batch->ssim_dc.p, ssim_weight, res_in.p, samples.scol.p, ctx->stream);
        SampleArgs a = args();
        a.in_res = res_in.p;
        launch_sample_raster(kVjp, a, ctx->stream);
        chain(nullptr, 0.f, dout);
        ctx->check_launch();
    }

    // b = J^T(-W r), r = render - truth at the samples (lm.cpp:99-121)
    void rhs_dev(float* dout) {
        launch_sample_raster(kRhs, args(), ctx->stream);
        chain(nullptr, 0.f, dout);
        ctx->check_launch();
    }

    void diag_dev(float* dout) {
        DiagArgs d{};
        d.groups = samples.groups.p;
        d.n_groups = static_cast<int>(samples.hgroups.size());
        d.cams = batch->cams.p;
        d.tile_offsets = batch->tile_offsets.p;
        d.entries = batch->entries.p;
        d.rec = batch->rec.p;
        d.Gp = scene->Gp;
        d.spix = samples.spix.p;
        d.sw = samples.sw.p;
        d.image = batch->image.p;
        d.last_img = batch->last.p;
        d.diagacc = diagacc.p;
        d.masks = samples.masks.p;
        d.glist = samples.glist.p;
        d.gcount = samples.gcount.p;
        d.mask_off = samples.mask_off.p;
        d.cols = samples.cols.p;
        d.scol = samples.scol.p;
        d.wbase = samples.wbase.p;
        d.partial = det ? samples.partial.p : nullptr;
        d.dest = samples.dest.p;
        launch_diag_raster(d, ctx->stream);
        launch_diag_finalize(scene->beta32.p, scene->G, scene->Gp, batch->cams.p, batch->V,
                             batch->conic.p, diagacc.p, det_order(), dout, ctx->stream);
        ctx->check_launch();
    }

    // ---- host-vector API (drop-in SampledJacobian methods)
    void upload_param(const double* h, float* d) {
        const int G = scene->G;
        host_stage.ensure(std::max<size_t>(static_cast<size_t>(kP) * G, 1));
        SLM_CUDA_CHECK(cudaMemsetAsync(d, 0, P() * sizeof(float), ctx->stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(host_stage.p, h, sizeof(double) * kP * G, cudaMemcpyHostToDevice, ctx->stream));
        launch_aos64_to_soa32(host_stage.p, G, scene->Gp, d, ctx->stream);
    }
    void download_param(const float* d, double* h) {
        const int G = scene->G;
        host_stage.ensure(std::max<size_t>(static_cast<size_t>(kP) * G, 1));
        launch_soa32_to_aos64(d, G, scene->Gp, host_stage.p, ctx->stream);
        SLM_CUDA_CHECK(cudaMemcpyAsync(h, host_stage.p, sizeof(double) * kP * G, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
    }

    void jvp(const double* v, double* out) {
        vin.ensure(P());
        res_out.ensure(std::max<long long>(rdim, 1));
        upload_param(v, vin.p);
        launch_tangents(scene->beta32.p, vin.p, scene->G, scene->Gp, batch->cams.p, batch->V, batch->conic.p,
                        tan.p, nullptr, ctx->stream);
        SampleArgs a = args();
        a.out_res = res_out.p;
        launch_sample_raster(kJvp, a, ctx->stream);
        ctx->check_launch();
        std::vector<float> h(rdim);
        SLM_CUDA_CHECK(cudaMemcpyAsync(h.data(), res_out.p, sizeof(float) * rdim, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        for (long long i = 0; i < rdim; ++i) out[i] = h[i];
    }

    void vjp(const double* uvec, double* out) {
        std::vector<float> h(rdim);
        for (long long i = 0; i < rdim; ++i) h[i] = static_cast<float>(uvec[i]);
        res_in.ensure(std::max<long long>(rdim, 1));
        vout.ensure(P());
        SLM_CUDA_CHECK(cudaMemcpyAsync(res_in.p, h.data(), sizeof(float) * rdim, cudaMemcpyHostToDevice, ctx->stream));
        SampleArgs a = args();
        a.in_res = res_in.p;
        launch_sample_raster(kVjp, a, ctx->stream);
        chain(nullptr, 0.f, vout.p);
        ctx->check_launch();
        download_param(vout.p, out);
    }

    void jtj_diag(double* out) {
        vout.ensure(P());
        diag_dev(vout.p);
        download_param(vout.p, out);
    }

    // The drop-in host-vector product (SampledJacobian::gn_apply): f64 AoS in and
    // out (the reference's ParamVector), pipelined in Gaussian chunks on a copy
    // stream: chunk c of p crosses PCIe while chunk c-1 is converted and its
    // tangents computed; after the raster, chunk c's result is converted and
    // copied back while chunk c+1's chain runs.  Per-Gaussian work only, so the
    // values are bitwise those of the unchunked product.  (Narrowing to f32 on
    // the host to halve the PCIe bytes measured slower: the host's memory
    // bandwidth, not PCIe, then bounds the call.)
    std::vector<cudaEvent_t> hev;
    cudaEvent_t hevent(size_t i) {
        while (hev.size() <= i) {
            cudaEvent_t e;
            SLM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            hev.push_back(e);
        }
        return hev[i];
    }
    ~Jacobian() {
        for (auto e : hev) cudaEventDestroy(e);
    }
    void gn_apply(double lambda, const double* pvec, double* out) {
        const int G = scene->G, Gp = scene->Gp;
        vin.ensure(P());
        vout.ensure(P());
        static const bool pipeline = [] {
            const char* e = std::getenv("SLM_HOST_PIPELINE");
            return !(e && e[0] == '0');
        }();
        if (ctx->world > 1 || G < 4096 || !pipeline) {  // small or sharded: one upload, one download
            upload_param(pvec, vin.p);
            gn_apply_dev(static_cast<float>(lambda), vin.p, vout.p);
            download_param(vout.p, out);
            return;
        }
        constexpr int kChunks = 8;
        const int step = round_up((G + kChunks - 1) / kChunks, 256);
        const int nch = (G + step - 1) / step;
        host_stage.ensure(static_cast<size_t>(kP) * G);
        cudaStream_t st = ctx->stream, cp = ctx->aux_stream();
        SLM_CUDA_CHECK(cudaMemsetAsync(vin.p, 0, P() * sizeof(float), st));  // padding Gaussians stay 0
        SLM_CUDA_CHECK(cudaEventRecord(hevent(0), st));
        SLM_CUDA_CHECK(cudaStreamWaitEvent(cp, hevent(0), 0));
        auto lo = [&](int c) { return c * step; };
        auto hi = [&](int c) { return std::min(G, (c + 1) * step); };
        for (int c = 0; c < nch; ++c) {
            const size_t a = static_cast<size_t>(kP) * lo(c), bytes = sizeof(double) * kP * (hi(c) - lo(c));
            SLM_CUDA_CHECK(cudaMemcpyAsync(host_stage.p + a, pvec + a, bytes, cudaMemcpyHostToDevice, cp));
            SLM_CUDA_CHECK(cudaEventRecord(hevent(1 + c), cp));
            SLM_CUDA_CHECK(cudaStreamWaitEvent(st, hevent(1 + c), 0));
            launch_aos64_to_soa32_range(host_stage.p, lo(c), hi(c), Gp, vin.p, st);
            launch_tangents_range(scene->beta32.p, vin.p, G, Gp, batch->cams.p, batch->V, batch->conic.p, tan.p,
                                  nullptr, lo(c), hi(c), st);
        }
        launch_sample_raster(kGn, args(), st);
        const float lam = static_cast<float>(lambda);
        for (int c = 0; c < nch; ++c) {
            launch_chain_range(scene->beta32.p, G, Gp, batch->cams.p, batch->V, batch->conic.p, inter.p, det_order(),
                               vin.p, lam, vout.p, nullptr, lo(c), hi(c), c == 0, st);
            launch_soa32_to_aos64_range(vout.p, lo(c), hi(c), Gp, host_stage.p, st);
            SLM_CUDA_CHECK(cudaEventRecord(hevent(1 + nch + c), st));
            SLM_CUDA_CHECK(cudaStreamWaitEvent(cp, hevent(1 + nch + c), 0));
            const size_t a = static_cast<size_t>(kP) * lo(c), bytes = sizeof(double) * kP * (hi(c) - lo(c));
            SLM_CUDA_CHECK(cudaMemcpyAsync(out + a, host_stage.p + a, bytes, cudaMemcpyDeviceToHost, cp));
        }
        ctx->check_launch();
        SLM_CUDA_CHECK(cudaStreamSynchronize(cp));
        SLM_CUDA_CHECK(cudaStreamSynchronize(st));
    }

    // pcg_solve (pcg.cpp:10-53) on device; returns the final CgState.
    CgState pcg_dev(float lambda, const float* b, const float* minv, int iters, float* x) {
        const size_t n = P();
        r.ensure(n);
        z.ensure(n);
        p.ensure(n);
        u.ensure(n);
        SLM_CUDA_CHECK(cudaMemsetAsync(u.p, 0, n * sizeof(float), ctx->stream));
        CgState* cg = ctx->cg.p;
        launch_cg_init(b, minv, static_cast<long long>(n), x, r.p, z.p, p.p, ctx->partial.p, cg, ctx->stream);
        for (int it = 0; it < iters; ++it) {
            gn_apply_dev(lambda, p.p, u.p, &cg->done);
            launch_cg_pu(p.p, u.p, static_cast<long long>(n), ctx->partial.p, cg, ctx->stream);
            launch_cg_update(x, r.p, z.p, p.p, u.p, minv, static_cast<long long>(n), ctx->partial.p, cg, ctx->stream);
        }
        ctx->check_launch();
        CgState h;
        SLM_CUDA_CHECK(cudaMemcpyAsync(&h, cg, sizeof(CgState), cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        return h;
    }
};

// =========================================================================== host samplers
// build_sample_plan (sample_plan.cpp:62-171) with libstdc++'s distributions.
struct PlanH {
    std::vector<int> view_camera;
    std::vector<int64_t> view_offset{0};
    std::vector<int> px, py, tile;
    std::vector<double> weight;
    int samples_per_tile = 0, dist = SLM_DIST_UNIFORM;
    slm_plan view() const {
        return slm_plan{static_cast<int32_t>(view_camera.size()), samples_per_tile, dist,
                        view_camera.data(), view_offset.data(), px.data(), py.data(), tile.data(),
                        weight.data()};
    }
    void clear() {
        view_camera.clear();
        view_offset.assign(1, 0);
        px.clear();
        py.clear();
        tile.clear();
        weight.clear();
    }
};

// Plans are recycled (their vectors keep their capacity): a fresh multi-MB
// allocation per LM step costs page faults on first touch that rival the
// sampler's own work at configs[0] (524k samples per step).
std::mutex g_plan_mu;
std::vector<std::unique_ptr<PlanH>> g_plan_pool;
static std::unique_ptr<PlanH> acquire_plan() {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    if (g_plan_pool.empty()) return std::make_unique<PlanH>();
    auto p = std::move(g_plan_pool.back());
    g_plan_pool.pop_back();
    p->clear();
    return p;
}
static void release_plan(std::unique_ptr<PlanH> p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_plan_mu);
    if (g_plan_pool.size() < 4) g_plan_pool.push_back(std::move(p));
}
struct PlanReturn {  // hands a step's plan back to the pool when the step ends
    std::unique_ptr<PlanH>& p;
    ~PlanReturn() { release_plan(std::move(p)); }
};

// Uniform plans with many samples (configs[0]: full pixels, 524k draws): the
// draws are libstdc++'s uniform_int_distribution<int>(i, m-1) on mt19937_64,
// i.e. Lemire's nearly-divisionless map (uniform_int_dist.h _S_nd): one 64-bit
// output x per draw gives i + (x * (m - i)) >> 64 unless the low half falls
// below (2^64 - r) % r (probability ~r / 2^64).  So the outputs are drawn
// sequentially (the RNG stream is the reference's) and the per-tile shuffles
// run on several threads; if any draw would have been rejected the whole plan
// is redone by the sequential reference loop from the saved RNG state.
// false: not handled (the caller runs the sequential loop).
static bool uniform_plan_parallel(PlanH* plan, const slm_camera* cams, int n_cams, int spt, size_t total,
                                  std::mt19937_64& rng) {
    struct TileJob {
        int x0, y0, rw, m, n, tile;
        size_t off;
    };
    std::vector<TileJob> jobs;
    std::vector<size_t> view_end;
    size_t off = 0;
    for (int ci = 0; ci < n_cams; ++ci) {
        const int txn = (cams[ci].width + kTile - 1) / kTile, tyn = (cams[ci].height + kTile - 1) / kTile;
        for (int ty = 0; ty < tyn; ++ty)
            for (int tx = 0; tx < txn; ++tx) {
                const int x0 = tx * kTile, y0 = ty * kTile;
                const int rw = std::min(cams[ci].width - x0, kTile), rh = std::min(cams[ci].height - y0, kTile);
                const int m = rw * rh, n = std::min(spt, m);
                jobs.push_back(TileJob{x0, y0, rw, m, n, ty * txn + tx, off});
                off += n;
            }
        view_end.push_back(off);
    }
    const std::mt19937_64 saved = rng;
    thread_local std::vector<uint64_t> raw;  // keeps its capacity (no first-touch faults per step)
    raw.resize(total);
    for (size_t k = 0; k < total; ++k) raw[k] = rng();
    plan->px.resize(total);
    plan->py.resize(total);
    plan->tile.resize(total);
    plan->weight.resize(total);
    const double n_total = static_cast<double>(total);
    const uint64_t* rawp = raw.data();  // (raw is this thread's thread_local: the workers get the pointer)
    std::atomic<bool> rejected{false};
    auto work = [&](size_t j0, size_t j1) {
        int pool[kTile * kTile];
        for (size_t j = j0; j < j1; ++j) {
            const TileJob& J = jobs[j];
            for (int l = 0; l < J.m; ++l) pool[l] = l;
            const uint64_t* x = rawp + J.off;
            for (int i = 0; i < J.n; ++i) {
                const uint64_t r = static_cast<uint64_t>(J.m - i);
                const unsigned __int128 prod = static_cast<unsigned __int128>(x[i]) * r;
                const uint64_t low = static_cast<uint64_t>(prod);
                if (low < r && low < (-r) % r) {  // _S_nd would draw again
                    rejected.store(true, std::memory_order_relaxed);
                    return;
                }
                std::swap(pool[i], pool[i + static_cast<int>(prod >> 64)]);
            }
            const double q = (J.n / n_total) * (1.0 / J.m);
            const double w = 1.0 / std::max(q, 1e-12);
            for (int i = 0; i < J.n; ++i) {
                plan->px[J.off + i] = J.x0 + pool[i] % J.rw;
                plan->py[J.off + i] = J.y0 + pool[i] / J.rw;
                plan->tile[J.off + i] = J.tile;
                plan->weight[J.off + i] = w;
            }
        }
    };
    const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency() / 2));
    std::vector<std::thread> th;
    const size_t per = (jobs.size() + nt - 1) / nt;
    for (unsigned t = 1; t < nt; ++t)
        if (t * per < jobs.size()) th.emplace_back(work, t * per, std::min(jobs.size(), (t + 1) * per));
    work(0, std::min(jobs.size(), per));
    for (auto& t : th) t.join();
    if (rejected.load()) {  // vanishingly rare: redo sequentially from the same RNG state
        rng = saved;
        plan->px.clear();
        plan->py.clear();
        plan->tile.clear();
        plan->weight.clear();
        return false;
    }
    for (int ci = 0; ci < n_cams; ++ci) {
        plan->view_camera.push_back(ci);
        plan->view_offset.push_back(static_cast<int64_t>(view_end[ci]));
    }
    return true;
}

static std::unique_ptr<PlanH> build_plan(const slm_camera* cams, int n_cams, int spt, int dist, int lane,
                                         std::mt19937_64& rng, const double* const* aux_image,
                                         const int32_t* const* aux_contrib, const double* const* aux_gt) {
    if (spt < 1) throw std::invalid_argument("samples_per_tile must be positive");
    if (spt > kTile * kTile) throw std::invalid_argument("samples_per_tile exceeds the pixels in a tile");
    if (lane < 1 || spt % lane != 0)
        throw std::invalid_argument("samples_per_tile must be a multiple of the lane width");
    if (dist != SLM_DIST_UNIFORM) {
        if (!aux_image || !aux_contrib) throw std::invalid_argument("weighted distributions need per-camera aux data");
        if (dist == SLM_DIST_RESIDUAL && !aux_gt)
            throw std::invalid_argument("residual distribution needs ground-truth images");
    }
    auto plan = acquire_plan();
    plan->samples_per_tile = spt;
    plan->dist = dist;
    size_t total = 0;
    for (int ci = 0; ci < n_cams; ++ci) {
        const int txn = (cams[ci].width + kTile - 1) / kTile, tyn = (cams[ci].height + kTile - 1) / kTile;
        for (int ty = 0; ty < tyn; ++ty)
            for (int tx = 0; tx < txn; ++tx) {
                const int w = std::min(cams[ci].width - tx * kTile, kTile);
                const int h = std::min(cams[ci].height - ty * kTile, kTile);
                total += std::min(spt, w * h);
            }
    }
    const double n_total = static_cast<double>(total);
    if (dist == SLM_DIST_UNIFORM && total >= (1u << 16) && uniform_plan_parallel(plan.get(), cams, n_cams, spt, total, rng))
        return plan;
    plan->px.reserve(total);
    plan->py.reserve(total);
    plan->tile.reserve(total);
    plan->weight.reserve(total);
    std::vector<int> pool;
    std::vector<double> density, cdf;
    for (int ci = 0; ci < n_cams; ++ci) {
        const slm_camera& cam = cams[ci];
        const int txn = (cam.width + kTile - 1) / kTile, tyn = (cam.height + kTile - 1) / kTile;
        plan->view_camera.push_back(ci);
        for (int ty = 0; ty < tyn; ++ty)
            for (int tx = 0; tx < txn; ++tx) {
                const int x0 = tx * kTile, y0 = ty * kTile;
                const int rw = std::min(cam.width - x0, kTile), rh = std::min(cam.height - y0, kTile);
                const int m = rw * rh, n = std::min(spt, m), tile = ty * txn + tx;
                auto emit = [&](int local, double q_tile) {
                    plan->px.push_back(x0 + local % rw);
                    plan->py.push_back(y0 + local / rw);
                    plan->tile.push_back(tile);
                    const double q = (n / n_total) * q_tile;
                    plan->weight.push_back(1.0 / std::max(q, 1e-12));
                };
                if (dist == SLM_DIST_UNIFORM) {
                    pool.resize(m);
                    std::iota(pool.begin(), pool.end(), 0);
                    for (int i = 0; i < n; ++i) {
                        std::uniform_int_distribution<int> d(i, m - 1);
                        std::swap(pool[i], pool[d(rng)]);
                    }
                    // emit(pool[i], 1.0 / m) with the per-tile constants hoisted: the
                    // weight is the same double expression for every sample of the tile
                    const double q = (n / n_total) * (1.0 / m);
                    const double w = 1.0 / std::max(q, 1e-12);
                    const size_t at = plan->px.size();
                    plan->px.resize(at + n);
                    plan->py.resize(at + n);
                    plan->tile.resize(at + n);
                    plan->weight.resize(at + n);
                    if (rw == kTile) {
                        for (int i = 0; i < n; ++i) {
                            plan->px[at + i] = x0 + (pool[i] & (kTile - 1));
                            plan->py[at + i] = y0 + (pool[i] >> 4);
                        }
                    } else {
                        for (int i = 0; i < n; ++i) {
                            plan->px[at + i] = x0 + pool[i] % rw;
                            plan->py[at + i] = y0 + pool[i] / rw;
                        }
                    }
                    std::fill(plan->tile.begin() + at, plan->tile.end(), tile);
                    std::fill(plan->weight.begin() + at, plan->weight.end(), w);
                    continue;
                }
                density.assign(m, 0.0);
                if (dist == SLM_DIST_RESIDUAL) {
                    double vmax = -1.0;
                    for (int l = 0; l < m; ++l) {
                        const size_t pix = static_cast<size_t>(y0 + l / rw) * cam.width + x0 + l % rw;
                        double v = 0.0;
                        for (int c = 0; c < 3; ++c) v += std::abs(aux_image[ci][3 * pix + c] - aux_gt[ci][3 * pix + c]);
                        density[l] = v / 3.0;
                        vmax = std::max(vmax, density[l]);
                    }
                    double sum = 0.0;
                    for (double& v : density) sum += (v = std::exp(v - vmax));
                    for (double& v : density) v /= sum;
                } else {
                    double sum = 0.0;
                    for (int l = 0; l < m; ++l) {
                        const size_t pix = static_cast<size_t>(y0 + l / rw) * cam.width + x0 + l % rw;
                        sum += (density[l] = 1.0 + aux_contrib[ci][pix]);
                    }
                    for (double& v : density) v /= sum;
                }
                cdf.resize(m);
                std::partial_sum(density.begin(), density.end(), cdf.begin());
                for (int k = 0; k < n; ++k) {
                    std::uniform_real_distribution<double> uni(0.0, 1.0);
                    const double uu = uni(rng) * cdf.back();
                    const auto it = std::upper_bound(cdf.begin(), cdf.end(), uu);
                    const int local = std::min<int>(static_cast<int>(it - cdf.begin()), m - 1);
                    emit(local, density[local]);
                }
            }
        plan->view_offset.push_back(static_cast<int64_t>(plan->px.size()));
    }
    return plan;
}

static std::unique_ptr<PlanH> exhaustive(const slm_camera* cams, int n_cams) {  // :173-197
    auto plan = std::make_unique<PlanH>();
    plan->samples_per_tile = kTile * kTile;
    double n_total = 0;
    for (int i = 0; i < n_cams; ++i) n_total += static_cast<double>(cams[i].width) * cams[i].height;
    for (int ci = 0; ci < n_cams; ++ci) {
        const int txn = (cams[ci].width + kTile - 1) / kTile;
        plan->view_camera.push_back(ci);
        for (int y = 0; y < cams[ci].height; ++y)
            for (int x = 0; x < cams[ci].width; ++x) {
                plan->px.push_back(x);
                plan->py.push_back(y);
                plan->tile.push_back((y / kTile) * txn + x / kTile);
                plan->weight.push_back(n_total);
            }
        plan->view_offset.push_back(static_cast<int64_t>(plan->px.size()));
    }
    return plan;
}

// camera_features / kmeans_cameras / sample_view_batch (view_sampler.cpp:10-184)
static std::vector<std::array<double, 6>> features(const slm_camera* cams, int n) {
    std::vector<std::array<double, 6>> f(n);
    if (n == 0) return f;
    double lo[3], hi[3];
    for (int i = 0; i < 3; ++i) {
        lo[i] = std::numeric_limits<double>::max();
        hi[i] = std::numeric_limits<double>::lowest();
    }
    std::vector<std::array<double, 3>> pos(n);
    for (int c = 0; c < n; ++c) {
        const double* r = cams[c].world_to_cam;
        const double* t = cams[c].translation;
        pos[c] = {-(r[0] * t[0] + r[3] * t[1] + r[6] * t[2]), -(r[1] * t[0] + r[4] * t[1] + r[7] * t[2]),
                  -(r[2] * t[0] + r[5] * t[1] + r[8] * t[2])};
        for (int i = 0; i < 3; ++i) {
            lo[i] = std::min(lo[i], pos[c][i]);
            hi[i] = std::max(hi[i], pos[c][i]);
        }
    }
    for (int c = 0; c < n; ++c) {
        for (int i = 0; i < 3; ++i) {
            const double ext = hi[i] - lo[i];
            f[c][i] = ext > 1e-12 ? (pos[c][i] - lo[i]) / ext : 0.5;
        }
        for (int i = 0; i < 3; ++i) f[c][3 + i] = cams[c].world_to_cam[6 + i];
    }
    return f;
}

static double dist6(const std::array<double, 6>& a, const std::array<double, 6>& b) {
    double acc = 0.0;
    for (int i = 0; i < 6; ++i) {
        const double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

static std::vector<int> kmeans(const std::vector<std::array<double, 6>>& f, int k, uint64_t seed) {
    const int n = static_cast<int>(f.size());
    if (k < 1) throw std::invalid_argument("cluster count must be at least 1");
    if (k > n) throw std::invalid_argument("cluster count exceeds camera count");
    std::mt19937_64 rng(seed);
    std::vector<std::array<double, 6>> cen;
    std::vector<bool> chosen(n, false);
    std::uniform_int_distribution<int> first(0, n - 1);
    const int idx = first(rng);
    cen.push_back(f[idx]);
    chosen[idx] = true;
    std::vector<double> d2(n);
    while (static_cast<int>(cen.size()) < k) {  // k-means++ seeding (:55-97)
        double total = 0.0;
        for (int i = 0; i < n; ++i) {
            d2[i] = std::numeric_limits<double>::max();
            for (const auto& c : cen) d2[i] = std::min(d2[i], dist6(f[i], c));
            if (chosen[i]) d2[i] = 0.0;
            total += d2[i];
        }
        int pick = -1;
        if (total > 0.0) {
            std::uniform_real_distribution<double> uni(0.0, total);
            double uu = uni(rng);
            for (int i = 0; i < n; ++i) {
                uu -= d2[i];
                if (uu <= 0.0) {
                    pick = i;
                    break;
                }
            }
            if (pick < 0) pick = n - 1;
        }
        if (pick < 0 || chosen[pick])
            pick = static_cast<int>(std::find(chosen.begin(), chosen.end(), false) - chosen.begin());
        cen.push_back(f[pick]);
        chosen[pick] = true;
    }
    std::vector<int> assign(n, -1);
    for (int iter = 0; iter < 100; ++iter) {  // Lloyd (:101-171)
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            int best = 0;
            double bd = dist6(f[i], cen[0]);
            for (int c = 1; c < k; ++c) {
                const double d = dist6(f[i], cen[c]);
                if (d < bd) {
                    bd = d;
                    best = c;
                }
            }
            if (assign[i] != best) {
                assign[i] = best;
                changed = true;
            }
        }
        std::vector<int> sizes(k, 0);
        for (int a : assign) ++sizes[a];
        for (int c = 0; c < k; ++c) {
            if (sizes[c] > 0) continue;
            int far = -1;
            double far_d = -1.0;
            for (int i = 0; i < n; ++i) {
                if (sizes[assign[i]] <= 1) continue;
                const double d = dist6(f[i], cen[assign[i]]);
                if (d > far_d) {
                    far_d = d;
                    far = i;
                }
            }
            if (far < 0) continue;
            --sizes[assign[far]];
            assign[far] = c;
            ++sizes[c];
            cen[c] = f[far];
            changed = true;
        }
        for (int c = 0; c < k; ++c) {
            std::array<double, 6> mean{};
            int count = 0;
            for (int i = 0; i < n; ++i) {
                if (assign[i] != c) continue;
                for (int d = 0; d < 6; ++d) mean[d] += f[i][d];
                ++count;
            }
            if (count > 0)
                for (int d = 0; d < 6; ++d) cen[c][d] = mean[d] / count;
        }
        if (!changed) break;
    }
    return assign;
}

static std::vector<int> view_batch(const std::vector<int>& assign, int k, std::mt19937_64& rng) {
    if (k < 1) throw std::invalid_argument("no clusters to sample from");
    std::vector<std::vector<int>> cl(k);
    for (size_t i = 0; i < assign.size(); ++i) {
        if (assign[i] < 0 || assign[i] >= k) throw std::invalid_argument("cluster index out of range");
        cl[assign[i]].push_back(static_cast<int>(i));
    }
    std::vector<int> batch;
    for (const auto& c : cl) {
        if (c.empty()) throw std::invalid_argument("empty cluster in batch sampler");
        std::uniform_int_distribution<size_t> d(0, c.size() - 1);
        batch.push_back(c[d(rng)]);
    }
    return batch;
}

// =========================================================================== TrainData + lm_step
struct Train {
    Context* ctx;
    std::vector<slm_camera> cams;
    std::vector<size_t> img_off;
    DevBuf<float> images;
    std::vector<int> assign;
    int k = 0;
};

static double learning_rate_from(double m, int iteration, const slm_lm_config& cfg) {  // lm.cpp:26-37
    if (iteration < cfg.warmup_iterations) return cfg.warmup_lr;
    if (m > 1.0) return std::min(cfg.lr_cap, 1.0 / m);
    return std::min(cfg.lr_cap, 1.0);
}

static void copy_gt(Train& t, Batch& b, const std::vector<int>& cam_ids) {
    b.gt.ensure(3 * std::max<long long>(b.n_pix, 1));
    for (size_t v = 0; v < cam_ids.size(); ++v) {
        const slm_camera& c = t.cams[cam_ids[v]];
        SLM_CUDA_CHECK(cudaMemcpyAsync(b.gt.p + 3 * b.hcams[v].pix_base, t.images.p + t.img_off[cam_ids[v]],
                                       sizeof(float) * 3 * c.width * c.height, cudaMemcpyDeviceToDevice,
                                       b.ctx->stream));
    }
}

// The next lm_step's view batch + sample plan + sample grouping, computed on a
// host thread while this step's PCG runs.  For the uniform distribution they
// depend only on the RNG state, the view clusters and the cameras, so the
// result is used iff the caller's RNG (and clusters, cameras, config) at the
// next call equal the snapshot taken here; otherwise it is discarded and the
// step draws as usual.  The RNG stream is the reference's either way.
struct Speculation {
    std::thread th;
    std::exception_ptr err;
    std::mt19937_64 rng_before, rng_after;
    std::vector<int> assign;
    int k = 0, spt = 0, dist = 0, lane = 0;
    std::vector<slm_camera> cams;
    std::vector<int> batch;
    std::unique_ptr<PlanH> plan;
    Jacobian* hj = nullptr;  // host half only (StepBuffers::spare)
    ~Speculation() {
        if (th.joinable()) th.join();
        release_plan(std::move(plan));
    }
};

struct StepBuffers {  // per-context persistent lm_step workspace (no per-step cudaMalloc)
    Batch batch;
    Jacobian jac;
    DevBuf<float> b, x, maxabs;
    Jacobian spare;  // host half of the speculated next step (vectors keep their pinned capacity)
    std::unique_ptr<Speculation> spec;
    explicit StepBuffers(Context* c) : batch(c), jac(c, nullptr, &batch), spare(c, nullptr, nullptr) {}
    ~StepBuffers() { spec.reset(); }
};

static bool same_cams(const std::vector<slm_camera>& a, const std::vector<slm_camera>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), sizeof(slm_camera) * a.size()) == 0);
}

void destroy_step(StepBuffers* s) { delete s; }

static StepBuffers& step_buffers(Context* ctx) {
    if (!ctx->step) ctx->step = new StepBuffers(ctx);
    return *ctx->step;
}

// ---- metrics (metrics/image_metrics.cpp, io/run.cpp:77-92) on device (metrics.cu)
static MetricWindow metric_window() {  // gaussian_window (image_metrics.cpp:25-35)
    MetricWindow w{};
    double sum = 0.0;
    for (int i = 0; i < kMetricWin; ++i) {
        const double d = i - kMetricWin / 2;
        w.w[i] = std::exp(-0.5 * d * d / (1.5 * 1.5));
        sum += w.w[i];
    }
    for (double& v : w.w) v /= sum;
    return w;
}

struct ImageRef {
    long long off;  // element offset of the interleaved RGB image
    int w, h;
};

// {sum of squared differences, sum of local SSIM} per image, both over the 3 channels.
// diag: metrics::ssim_diag_residuals mode ({sse, sum of s^2}; planes when res != nullptr).
template <typename T>
static std::vector<double2> image_metrics(Context* c, const T* a, const T* b, const std::vector<ImageRef>& imgs,
                                          bool diag = false, T* res = nullptr, T* dcen = nullptr) {
    const int n = static_cast<int>(imgs.size());
    std::vector<ImgDesc> hd(n);
    int base = 0, max_tiles = 0;
    for (int i = 0; i < n; ++i) {
        ImgDesc& d = hd[i];
        d.off = imgs[i].off;
        d.w = imgs[i].w;
        d.h = imgs[i].h;
        d.tiles = metric_tiles(d.w, d.h, &d.tiles_x);
        d.tile_base = base;
        base += d.tiles;
        max_tiles = std::max(max_tiles, d.tiles);
    }
    std::vector<double2> out(n);
    if (n == 0) return out;
    DevBuf<ImgDesc> dd;
    DevBuf<double2> part, dout;
    dd.ensure(n);
    part.ensure(std::max(base, 1));
    dout.ensure(n);
    SLM_CUDA_CHECK(cudaMemcpyAsync(dd.p, hd.data(), sizeof(ImgDesc) * n, cudaMemcpyHostToDevice, c->stream));
    if (diag)
        launch_ssim_diag(a, b, dd.p, n, max_tiles, part.p, dout.p, metric_window(), res, dcen, c->stream);
    else
        launch_image_metrics(a, b, dd.p, n, max_tiles, part.p, dout.p, metric_window(), c->stream);
    c->check_launch();
    SLM_CUDA_CHECK(cudaMemcpyAsync(out.data(), dout.p, sizeof(double2) * n, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return out;
}

// metrics::evaluate (image_metrics.cpp:180-186) from the device sums.
// Per view {sse, sum of s^2} of the batch render vs truth
// (metrics::ssim_diag_residuals); with planes, B.ssim_res / B.ssim_dc get s and
// ds/dcentre per pixel and channel.
// exact: of the FP64 render (k_render_exact) vs the widened truth, as the
// reference computes them (lm.cpp:39-54,86-119 on render_full's f64 image);
// the planes are then narrowed to f32 for the products.
static std::vector<double2> batch_ssim(Batch& B, bool planes, bool exact = false) {
    std::vector<ImageRef> imgs;
    for (int v = 0; v < B.V; ++v) imgs.push_back({3 * B.hcams[v].pix_base, B.hcams[v].width, B.hcams[v].height});
    const long long n3 = 3 * std::max<long long>(B.n_pix, 1);
    if (planes) {
        B.ssim_res.ensure(n3);
        B.ssim_dc.ensure(n3);
    }
    if (!exact)
        return image_metrics<float>(B.ctx, B.image.p, B.gt.p, imgs, true, planes ? B.ssim_res.p : nullptr,
                                    planes ? B.ssim_dc.p : nullptr);
    B.render_exact();
    B.widen_gt();
    if (planes) {
        B.ssim_res64.ensure(n3);
        B.ssim_dc64.ensure(n3);
    }
    auto out = image_metrics<double>(B.ctx, B.image64.p, B.gt64.p, imgs, true, planes ? B.ssim_res64.p : nullptr,
                                     planes ? B.ssim_dc64.p : nullptr);
    if (planes) {
        launch_narrow(B.ssim_res64.p, B.ssim_res.p, 3 * B.n_pix, B.ctx->stream);
        launch_narrow(B.ssim_dc64.p, B.ssim_dc.p, 3 * B.n_pix, B.ctx->stream);
        B.ctx->check_launch();
    }
    return out;
}

constexpr int kEvalChunk = 8;  // cameras per device batch outside lm_step (bounds the batch buffers)

// batch_loss (lm.cpp:39-54) over the given TrainData cameras, on the device.
static double batch_loss_dev(Scene& s, Train& t, const std::vector<int>& ids, int loss, double ssim_weight,
                             Batch& b) {
    if (loss != SLM_LOSS_MSE && loss != SLM_LOSS_MSE_SSIM) throw std::invalid_argument("batch_loss: unknown loss");
    double acc = 0.0;
    for (size_t lo = 0; lo < ids.size(); lo += kEvalChunk) {
        const size_t hi = std::min(ids.size(), lo + kEvalChunk);
        std::vector<int> chunk(ids.begin() + lo, ids.begin() + hi);
        std::vector<slm_camera> cv;
        for (int i : chunk) {
            if (i < 0 || i >= static_cast<int>(t.cams.size())) throw std::invalid_argument("camera index");
            cv.push_back(t.cams[i]);
        }
        b.prepare(s, cv);
        copy_gt(t, b, chunk);
        b.render(true, false);
        auto sse = b.view_sse();
        std::vector<double2> ss;
        if (loss == SLM_LOSS_MSE_SSIM) {  // both terms of the FP64 render, like the reference's
            ss = batch_ssim(b, false, true);
            for (int v = 0; v < b.V; ++v) sse[v] = ss[v].x;
        }
        for (int v = 0; v < b.V; ++v) {
            const double n3 = 3.0 * cv[v].width * cv[v].height;
            double term = sse[v] / n3;
            if (loss == SLM_LOSS_MSE_SSIM) term += ssim_weight * ss[v].y / n3;
            acc += term;
        }
    }
    return ids.empty() ? 0.0 : acc / static_cast<double>(ids.size());
}

// baselines::full_gradient (first_order.cpp:11-44) over every TrainData camera:
// exhaustive plan, u = 2/M (r + w s s'), J^T u, accumulated over camera chunks
// into grad (f32 SoA [14][Gp]).
static void full_gradient_dev(Scene& s, Train& t, int loss, double ssim_weight, Batch& B, Jacobian& J,
                              DevBuf<float>& chunk, float* grad) {
    if (loss != SLM_LOSS_MSE && loss != SLM_LOSS_MSE_SSIM) throw std::invalid_argument("full_gradient: unknown loss");
    Context* ctx = s.ctx;
    const size_t P = s.P();
    chunk.ensure(P);
    SLM_CUDA_CHECK(cudaMemsetAsync(grad, 0, P * sizeof(float), ctx->stream));
    double entries = 0.0;
    for (const auto& c : t.cams) entries += 3.0 * c.width * c.height;
    const float scale = static_cast<float>(2.0 / entries);
    J.scene = &s;
    for (size_t lo = 0; lo < t.cams.size(); lo += kEvalChunk) {
        const size_t hi = std::min(t.cams.size(), lo + kEvalChunk);
        std::vector<int> ids;
        std::vector<slm_camera> cv;
        for (size_t i = lo; i < hi; ++i) {
            ids.push_back(static_cast<int>(i));
            cv.push_back(t.cams[i]);
        }
        B.prepare(s, cv);
        copy_gt(t, B, ids);
        B.render(false, false);
        if (loss == SLM_LOSS_MSE_SSIM) batch_ssim(B, true);
        J.init_host_exhaustive(cv, loss == SLM_LOSS_MSE_SSIM ? B.ssim_res.p : nullptr, B.ssim_dc.p,
                               static_cast<float>(ssim_weight), scale);
        J.init_device();
        SampleArgs a = J.args();
        a.in_res = J.res_in.p;
        launch_sample_raster(kVjp, a, ctx->stream);
        J.chain(nullptr, 0.f, chunk.p);
        launch_axpy(grad, chunk.p, static_cast<long long>(P), 1.0f, ctx->stream);
        ctx->check_launch();
    }
}

// first_order_step (first_order.cpp:54-122) parameters for step number `step` (1-based after ++).
static FirstOrderParams first_order_params(const slm_first_order_config& c, long long step) {
    if (c.kind < SLM_FO_ADAM || c.kind > SLM_FO_SGD_MOMENTUM) throw std::invalid_argument("unknown first-order optimizer");
    FirstOrderParams fp{};
    fp.kind = c.kind;
    double mean_factor = 1.0;  // mean_lr_factor(cfg, step - 1) (:54-58)
    if (c.decay_iterations > 0) {
        const double t = std::min(1.0, static_cast<double>(step - 1) / c.decay_iterations);
        mean_factor = std::pow(c.mean_lr_final_factor, t);
    }
    for (int k = 0; k < kP; ++k) {  // group_lr (:46-52)
        double lr = k < 3 ? c.lr_mean : k < 6 ? c.lr_scale : k < 10 ? c.lr_rotation : k == 10 ? c.lr_opacity : c.lr_color;
        if (k < 3) lr *= mean_factor;
        fp.lr[k] = lr;
    }
    if (c.kind == SLM_FO_ADAM) {
        fp.b1 = c.adam_beta1;
        fp.b2 = c.adam_beta2;
        fp.eps = c.adam_eps;
        fp.c1 = 1.0 - std::pow(c.adam_beta1, static_cast<double>(step));
        fp.c2 = 1.0 - std::pow(c.adam_beta2, static_cast<double>(step));
    } else if (c.kind == SLM_FO_RMSPROP) {
        fp.b2 = c.rms_decay;
        fp.eps = c.rms_eps;
    } else {
        fp.b1 = c.momentum;
    }
    return fp;
}

// FirstOrderState (first_order.hpp:39-51) on the device + the workspaces of
// full_gradient and batch_loss.
struct FirstOrder {
    Scene* scene;
    DevBuf<double> m1, m2, g64;
    long long step = 0;
    Batch batch;
    Jacobian jac;
    DevBuf<float> grad, chunk;
    FirstOrder(const FirstOrder&) = delete;
    FirstOrder& operator=(const FirstOrder&) = delete;
    explicit FirstOrder(Scene* s) : scene(s), batch(s->ctx), jac(s->ctx, s, &batch) {
        const size_t P = s->P();
        m1.ensure(P);
        m2.ensure(P);
        SLM_CUDA_CHECK(cudaMemsetAsync(m1.p, 0, P * sizeof(double), s->ctx->stream));
        SLM_CUDA_CHECK(cudaMemsetAsync(m2.p, 0, P * sizeof(double), s->ctx->stream));
    }
    void apply(const float* g32, const double* g64_aos, const slm_first_order_config& c) {
        const FirstOrderParams fp = first_order_params(c, step + 1);
        ++step;
        launch_first_order_step(scene->beta.p, scene->beta32.p, m1.p, m2.p, g32, g64_aos, scene->G, scene->Gp, fp,
                                scene->ctx->stream);
        scene->ctx->check_launch();
    }
};

static slm_metric_report metric_report(double2 s, int w, int h) {
    slm_metric_report r{};
    const double n = static_cast<double>(w) * h;
    r.mse = n == 0 ? 0.0 : s.x / (3.0 * n);                  // :108-113
    r.psnr = r.mse < 1e-10 ? 100.0 : 10.0 * std::log10(1.0 / r.mse);  // :115-119
    r.ssim = n == 0 ? 1.0 : s.y / (3.0 * n);                 // :121-139
    return r;
}
static void lm_step(Scene& s, Train& t, const slm_lm_config& cfg, int iteration, std::mt19937_64& rng,
                    slm_step_report& rep) {
    Context* ctx = s.ctx;
    ctx->activate();
    if (t.k < 1) throw std::invalid_argument("lm_step: no view clusters");
    if (cfg.loss != SLM_LOSS_MSE && cfg.loss != SLM_LOSS_MSE_SSIM) throw std::invalid_argument("lm_step: unknown loss");
    const bool ssim = cfg.loss == SLM_LOSS_MSE_SSIM;
    ctx->mark("start");
    rep.iteration = iteration;
    StepBuffers& sb = step_buffers(ctx);
    // the previous step's speculative draw of this step's batch + plan (see Speculation)
    std::unique_ptr<Speculation> spec = std::move(sb.spec);
    bool use_spec = false;
    if (spec) {
        if (spec->th.joinable()) spec->th.join();
        use_spec = !spec->err && spec->rng_before == rng && spec->k == t.k &&
                   spec->assign == t.assign && spec->spt == cfg.samples_per_tile && spec->dist == cfg.dist &&
                   spec->lane == cfg.sample_lane_width && same_cams(spec->cams, t.cams);
    }
    // 1. view batch (lm.cpp:63)
    const std::vector<int> batch = use_spec ? spec->batch : view_batch(t.assign, t.k, rng);
    const int VB = static_cast<int>(batch.size());
    int lo = 0, hi = 0;
    slm_view_slice(VB, ctx->rank, ctx->world, &lo, &hi);
    std::vector<slm_camera> all_cams, my_cams;
    std::vector<int> my_ids;
    for (int i = 0; i < VB; ++i) all_cams.push_back(t.cams[batch[i]]);
    for (int i = lo; i < hi; ++i) {
        my_cams.push_back(t.cams[batch[i]]);
        my_ids.push_back(batch[i]);
    }
    Batch& B = sb.batch;
    Jacobian& J = sb.jac;
    J.scene = &s;
    // 4. (host) plan for the whole batch — every rank replays the same RNG
    // stream (sample_plan.cpp:62-171) — and the sample grouping.  For the
    // uniform distribution the plan does not depend on the render, so it runs
    // on a host thread while the GPU prepares and renders the views.
    std::unique_ptr<PlanH> plan;
    PlanReturn plan_return{plan};
    std::exception_ptr plan_err;
    auto make_plan = [&] {
        try {
            plan = build_plan(all_cams.data(), VB, cfg.samples_per_tile, cfg.dist, cfg.sample_lane_width, rng,
                              nullptr, nullptr, nullptr);
            const long long total = plan->view_offset.back();
            J.init_host(plan->view(), lo, hi, total > 0 ? 1.0 / static_cast<double>(total) : 0.0, my_cams);
        } catch (...) {
            plan_err = std::current_exception();
        }
    };
    // Weighted distributions: the host draws the uniforms (the whole RNG
    // consumption of the plan), the device picks the pixels from the render
    // (Jacobian::Draw) -- so this overlaps with the render too.
    auto make_weighted = [&] {
        try {
            J.init_host_weighted(all_cams, lo, hi, cfg.samples_per_tile, cfg.dist, cfg.sample_lane_width, rng);
        } catch (...) {
            plan_err = std::current_exception();
        }
    };
    std::thread sampler;
    if (use_spec) {
        plan = std::move(spec->plan);
        J.take_host(*spec->hj);
        rng = spec->rng_after;
    } else if (cfg.dist == SLM_DIST_UNIFORM) {
        sampler = std::thread(make_plan);
    } else {
        sampler = std::thread(make_weighted);
    }
    spec.reset();
    // 2./3. forward render + residual fields of this rank's views (lm.cpp:75-78)
    try {
        B.prepare(s, my_cams);
        copy_gt(t, B, my_ids);
        B.render(true, false);
    } catch (...) {
        if (sampler.joinable()) sampler.join();
        throw;
    }
    ctx->mark("prepare+render");
    if (sampler.joinable()) sampler.join();
    ctx->mark("plan:host");
    if (plan_err) std::rethrow_exception(plan_err);
    {  // speculate the next step's batch + plan (uniform) or uniforms (weighted) while this one
       // solves: started as soon as this step's draws are final, so the host draw of a
       // full-pixel plan (configs[0]: 524k samples) hides behind the whole step
        auto sp = std::make_unique<Speculation>();
        sp->rng_before = rng;
        sp->assign = t.assign;
        sp->k = t.k;
        sp->spt = cfg.samples_per_tile;
        sp->dist = cfg.dist;
        sp->lane = cfg.sample_lane_width;
        sp->cams = t.cams;
        sp->hj = &sb.spare;
        Speculation* q = sp.get();
        const int rank = ctx->rank, world = ctx->world;
        q->th = std::thread([q, rank, world] {
            try {
                std::mt19937_64 r = q->rng_before;
                q->batch = view_batch(q->assign, q->k, r);
                const int nb = static_cast<int>(q->batch.size());
                int l = 0, h = 0;
                slm_view_slice(nb, rank, world, &l, &h);
                std::vector<slm_camera> all, mine;
                for (int i = 0; i < nb; ++i) all.push_back(q->cams[q->batch[i]]);
                for (int i = l; i < h; ++i) mine.push_back(q->cams[q->batch[i]]);
                if (q->dist == SLM_DIST_UNIFORM) {
                    q->plan = build_plan(all.data(), nb, q->spt, q->dist, q->lane, r, nullptr, nullptr, nullptr);
                    const long long total = q->plan->view_offset.back();
                    q->hj->init_host(q->plan->view(), l, h, total > 0 ? 1.0 / static_cast<double>(total) : 0.0,
                                     mine);
                } else {
                    q->hj->init_host_weighted(all, l, h, q->spt, q->dist, q->lane, r);
                }
                q->rng_after = r;
            } catch (...) {
                q->err = std::current_exception();
            }
        });
        sb.spec = std::move(sp);
    }
    J.upload_early();  // overlaps the render still running on the main stream
    // loss_before: mean of the per-view MSE of the pre-update renders (lm.cpp:143-147)
    double before = 0.0;
    if (ssim) {  // mse + ssim_weight * mean s^2 per view (lm.cpp:143-147) of the FP64 render; planes for the rhs fold
        const auto ss = batch_ssim(B, true, true);
        for (int v = 0; v < B.V; ++v)
            before += (ss[v].x + cfg.ssim_weight * ss[v].y) / (3.0 * my_cams[v].width * my_cams[v].height);
        ctx->mark("ssim");
    } else {
        const auto sse = B.view_sse();
        for (int v = 0; v < B.V; ++v)
            before += sse[v] / (3.0 * my_cams[v].width * my_cams[v].height);
    }
    J.init_device();
    ctx->mark("plan");
    const size_t P = s.P();
    sb.b.ensure(2 * P);  // [b | diag] contiguous for one fused allreduce
    sb.x.ensure(P);
    sb.maxabs.ensure(1);
    float* db = sb.b.p;
    float* dd = sb.b.p + P;
    SLM_CUDA_CHECK(cudaMemsetAsync(sb.b.p, 0, 2 * P * sizeof(float), ctx->stream));
    // 5. b = J^T(-W r) and diag(J^T W J) (lm.cpp:121-125)
    if (ssim)
        J.rhs_ssim_dev(db, static_cast<float>(cfg.ssim_weight));
    else
        J.rhs_dev(db);
    ctx->mark("rhs");
    J.diag_dev(dd);
    ctx->allreduce(sb.b.p, 2 * P);
    launch_minv(dd, static_cast<long long>(P), static_cast<float>(cfg.damping), ctx->stream);
    ctx->mark("diag");
    // 7. PCG (lm.cpp:128-132)
    const int iters = iteration >= cfg.pcg_switch_iteration ? cfg.pcg_iters_late : cfg.pcg_iters_initial;
    const CgState cs = J.pcg_dev(static_cast<float>(cfg.damping), db, dd, iters, sb.x.p);
    rep.pcg_iterations = cs.iterations;
    rep.breakdown = cs.breakdown;
    ctx->mark("pcg");
    ctx->step_stats[0] = B.V;
    ctx->step_stats[1] = std::accumulate(B.valid_count.begin(), B.valid_count.end(), 0ll);
    ctx->step_stats[2] = B.n_entries;
    ctx->step_stats[3] = J.samples.total;
    ctx->step_stats[4] = B.n_pix;
    ctx->step_stats[5] = cs.iterations;
    // 8./9./10. learning rate and update (lm.cpp:135-137)
    launch_color_maxabs(sb.x.p, s.G, s.Gp, sb.maxabs.p, ctx->stream);
    float m = 0.f;
    SLM_CUDA_CHECK(cudaMemcpyAsync(&m, sb.maxabs.p, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    rep.eta = learning_rate_from(static_cast<double>(m), iteration, cfg);
    if (cs.breakdown) rep.eta *= 0.5;
    launch_apply_update(s.beta.p, sb.x.p, s.G, s.Gp, rep.eta, s.beta32.p, ctx->stream);
    ctx->check_launch();
    ctx->mark("update");
    // loss_after = batch_loss of the updated state (lm.cpp:149-153)
    B.prepare(s, my_cams, ssim);  // mse+ssim: both terms come from the FP64 render
    B.render(true, false);
    ctx->step_stats[6] = std::accumulate(B.valid_count.begin(), B.valid_count.end(), 0ll);
    ctx->step_stats[7] = B.n_entries;
    double after = 0.0;
    {
        auto sse = B.view_sse();
        std::vector<double2> ss;
        if (ssim) {  // both terms of the FP64 render (batch_loss, lm.cpp:44-50)
            ss = batch_ssim(B, false, true);
            for (int v = 0; v < B.V; ++v) sse[v] = ss[v].x;
        }
        for (int v = 0; v < B.V; ++v) {
            const double n3 = 3.0 * my_cams[v].width * my_cams[v].height;
            double term = sse[v] / n3;
            if (ssim) term += cfg.ssim_weight * ss[v].y / n3;
            after += term;
        }
    }
    if (ctx->world > 1) {
        double h[2] = {before, after};
        ctx->dscalar.ensure(2);
        SLM_CUDA_CHECK(cudaMemcpyAsync(ctx->dscalar.p, h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
        ctx->allreduce(ctx->dscalar.p, 2);
        SLM_CUDA_CHECK(cudaMemcpyAsync(h, ctx->dscalar.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->sync();
        before = h[0];
        after = h[1];
    }
    ctx->mark("loss_after");
    ctx->finish_marks();
    rep.loss_before = before / VB;
    rep.loss_after = after / VB;
    rep.batch_size = VB;
    for (int i = 0; i < VB && i < rep.batch_capacity; ++i) rep.batch[i] = batch[i];
    if (!std::isfinite(rep.loss_after)) throw std::runtime_error("lm_step: non-finite loss after update");
}

}  // namespace slm

// =========================================================================== C ABI
using namespace slm;

struct slm_context { Context impl; explicit slm_context(int d) : impl(d) {} };
struct slm_scene { Scene impl; slm_scene(Context* c, const slm_gaussians& h) : impl(c, h) {} };
struct slm_rng { std::mt19937_64 eng; explicit slm_rng(uint64_t s) : eng(s) {} };
struct slm_plan_h { std::unique_ptr<PlanH> impl; };
struct slm_train { Train impl; };
struct slm_jacobian {
    std::unique_ptr<Scene> scene;
    std::unique_ptr<Batch> batch;
    std::unique_ptr<Jacobian> jac;
};

namespace {
template <class F>
int guarded(F&& f) {
    try {
        f();
        return SLM_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SLM_E_INVALID;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SLM_E_DOMAIN;
    } catch (const CudaError& e) {
        g_err = e.what();
        return SLM_E_CUDA;
    } catch (const NcclError& e) {
        g_err = e.what();
        return SLM_E_CUDA;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return SLM_E_RUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SLM_E_RUNTIME;
    }
}

Jacobian* make_jacobian(Context* ctx, Scene* scene, const slm_camera* cams, int n_cams, const slm_plan& plan,
                        slm_jacobian* holder) {
    std::vector<slm_camera> vc;
    for (int v = 0; v < plan.n_views; ++v) {
        if (plan.view_camera[v] < 0 || plan.view_camera[v] >= n_cams)
            throw std::invalid_argument("sample plan references a camera outside the batch");
        vc.push_back(cams[plan.view_camera[v]]);
    }
    holder->batch = std::make_unique<Batch>(ctx);
    holder->batch->prepare(*scene, vc);
    holder->batch->render(false);
    holder->jac = std::make_unique<Jacobian>(ctx, scene, holder->batch.get());
    const long long total = plan.view_offset[plan.n_views];
    holder->jac->init_host(plan, 0, plan.n_views, total > 0 ? 1.0 / static_cast<double>(total) : 0.0, vc);
    holder->jac->init_device();
    ctx->sync();
    return holder->jac.get();
}
}  // namespace

extern "C" {

const char* slm_last_error(void) { return g_err.c_str(); }
int slm_version(void) { return 1; }
int slm_device_count(int* out) {
    return guarded([&] { SLM_CUDA_CHECK(cudaGetDeviceCount(out)); });
}

int slm_context_create(int device, slm_context** out) {
    *out = nullptr;
    return guarded([&] { *out = new slm_context(device); });
}
int slm_context_destroy(slm_context* ctx) {
    return guarded([&] { delete ctx; });
}
int slm_context_synchronize(slm_context* ctx) {
    return guarded([&] { ctx->impl.sync(); });
}
int slm_context_set_stream(slm_context* ctx, void* stream) {
    return guarded([&] {
        Context& c = ctx->impl;
        if (c.stream && c.own_stream) cudaStreamDestroy(c.stream);
        c.stream = static_cast<cudaStream_t>(stream);
        c.own_stream = false;
    });
}
int slm_context_last_samples(slm_context* ctx, int64_t capacity, int64_t* n, int32_t* px, int32_t* py,
                              float* weight) {
    return guarded([&] {
        Context& c = ctx->impl;
        if (!c.step) throw std::invalid_argument("no lm_step has run on this context");
        Samples& S = c.step->jac.samples;
        const long long total = S.total;
        *n = total;
        if (capacity < total || total == 0) return;
        std::vector<int> pix(total), orig(total);
        std::vector<float> w(3 * total);
        c.activate();
        SLM_CUDA_CHECK(cudaMemcpyAsync(pix.data(), S.spix.p, sizeof(int) * total, cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(orig.data(), S.sorig.p, sizeof(int) * total, cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(w.data(), S.sw.p, sizeof(float) * 3 * total, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (long long k = 0; k < total; ++k) {  // group order -> plan order (view, tile, draw)
            const long long o = orig[k];
            if (o < 0 || o >= total) throw std::runtime_error("sample order out of range");
            px[o] = pix[k] & 0xffff;
            py[o] = pix[k] >> 16;
            weight[o] = w[3 * k];
        }
    });
}
int slm_context_step_stats(slm_context* ctx, int64_t out[8]) {
    return guarded([&] {
        for (int i = 0; i < 8; ++i) out[i] = ctx->impl.step_stats[i];
    });
}
int slm_context_set_comm_chunks(slm_context* ctx, int chunks) {
    return guarded([&] {
        if (chunks < 1) throw std::invalid_argument("comm chunks must be positive");
        ctx->impl.comm_chunks = chunks;
    });
}
int slm_context_set_deterministic(slm_context* ctx, int on) {
    return guarded([&] { ctx->impl.deterministic = on != 0; });
}
int slm_context_set_timing(slm_context* ctx, int on) {
    return guarded([&] { ctx->impl.timing = on != 0; });
}
int slm_context_timings(slm_context* ctx, double* out, int capacity, int* n) {
    return guarded([&] {
        const auto& t = ctx->impl.last_timings;
        *n = static_cast<int>(t.size());
        for (int i = 0; i < *n && i < capacity; ++i) out[i] = t[i];
    });
}
long long slm_launch_count(void) { return g_launches.load(); }
const char* slm_context_timing_names(slm_context* ctx) { return ctx->impl.last_timing_names.c_str(); }
int slm_context_set_profiling(slm_context* ctx, int on) {
    return guarded([&] { ctx->impl.prof = on != 0; });
}
int slm_context_profile_collect(slm_context* ctx, double out[3], int* n) {
    return guarded([&] { ctx->impl.prof_collect(out, n); });
}

int slm_nccl_unique_id(uint8_t out[128]) {
    return guarded([&] {
        ncclUniqueId id;
        SLM_NCCL_CHECK(nccl().GetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(out, &id, 128);
    });
}
int slm_context_init_comm(slm_context* ctx, const uint8_t id[128], int rank, int world) {
    return guarded([&] {
        Context& c = ctx->impl;
        c.activate();
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
        c.comm.reset();
        if (world > 1) {
            ncclUniqueId uid;
            std::memcpy(&uid, id, 128);
            auto nc = std::make_unique<NcclComm>();
            SLM_NCCL_CHECK(nccl().CommInitRank(&nc->c, world, uid, rank));
            c.comm = std::move(nc);
        }
        c.rank = rank;
        c.world = world;
    });
}
struct slm_local_group {
    std::shared_ptr<LocalGroup> g;
};
int slm_local_group_create(int world, slm_local_group** out) {
    return guarded([&] {
        if (world < 1 || world > 64) throw std::invalid_argument("local group: world must be in [1, 64]");
        *out = new slm_local_group{std::make_shared<LocalGroup>(world)};
    });
}
void slm_local_group_destroy(slm_local_group* g) { delete g; }
int slm_context_init_local(slm_context* ctx, slm_local_group* group, int rank) {
    return guarded([&] {
        Context& c = ctx->impl;
        c.activate();
        const int world = group->g->world;
        if (rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
        c.comm.reset();
        if (world > 1) c.comm = std::make_unique<LocalComm>(group->g, rank, c.device);
        c.rank = rank;
        c.world = world;
    });
}
int slm_context_rank(slm_context* ctx, int* rank, int* world) {
    *rank = ctx->impl.rank;
    *world = ctx->impl.world;
    return SLM_OK;
}

int slm_rng_create(uint64_t seed, slm_rng** out) {
    return guarded([&] { *out = new slm_rng(seed); });
}
void slm_rng_destroy(slm_rng* rng) { delete rng; }
uint64_t slm_rng_next(slm_rng* rng) { return rng->eng(); }
// std::mt19937_64 state as libstdc++'s operator<< text (312 words + index):
// lets a C++ caller hand its own engine to lm_step across the C ABI.
int slm_rng_get_state(slm_rng* rng, char* buf, int64_t capacity, int64_t* length) {
    return guarded([&] {
        std::ostringstream os;
        os << rng->eng;
        const std::string str = os.str();
        *length = static_cast<int64_t>(str.size());
        if (capacity > static_cast<int64_t>(str.size())) std::memcpy(buf, str.c_str(), str.size() + 1);
    });
}
int slm_rng_set_state(slm_rng* rng, const char* text) {
    return guarded([&] {
        std::istringstream is(text);
        is >> rng->eng;
        if (is.fail()) throw std::invalid_argument("malformed mt19937_64 state");
    });
}
// The contiguous view slice rank `rank` of `world` owns in a batch of n views.
int slm_view_slice(int n, int rank, int world, int* lo, int* hi) {
    if (world < 1 || rank < 0 || rank >= world || n < 0) return SLM_E_INVALID;
    *lo = static_cast<int>(static_cast<long long>(n) * rank / world);
    *hi = static_cast<int>(static_cast<long long>(n) * (rank + 1) / world);
    return SLM_OK;
}

int slm_scene_create(slm_context* ctx, const slm_gaussians* host, slm_scene** out) {
    return guarded([&] {
        ctx->impl.activate();
        *out = new slm_scene(&ctx->impl, *host);
        ctx->impl.sync();
    });
}
void slm_scene_destroy(slm_scene* s) { delete s; }
int slm_scene_upload(slm_scene* s, const slm_gaussians* host) {
    return guarded([&] {
        s->impl.upload(*host);
        s->impl.ctx->sync();
    });
}
int slm_scene_download(slm_scene* s, slm_gaussians* host) {
    return guarded([&] { s->impl.download(*host); });
}
int slm_scene_count(slm_scene* s, int* count, int* padded) {
    *count = s->impl.G;
    *padded = s->impl.Gp;
    return SLM_OK;
}
int slm_scene_apply_update(slm_scene* s, const double* delta_aos, double eta) {
    return guarded([&] {
        Scene& sc = s->impl;
        Context* c = sc.ctx;
        c->activate();
        DevBuf<double> d;
        d.ensure(std::max<size_t>(static_cast<size_t>(kP) * sc.G, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(d.p, delta_aos, sizeof(double) * kP * sc.G, cudaMemcpyHostToDevice, c->stream));
        launch_apply_update_f64(sc.beta.p, d.p, sc.G, sc.Gp, eta, sc.beta32.p, c->stream);
        c->check_launch();
        c->sync();
    });
}
int slm_scene_beta_ptrs(slm_scene* s, double** beta, float** beta32) {
    *beta = s->impl.beta.p;
    *beta32 = s->impl.beta32.p;
    return SLM_OK;
}

int slm_bin_and_sort(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam, int32_t* offsets,
                     int32_t* indices, int64_t capacity, int64_t* n_entries) {
    return guarded([&] {
        Context* c = &ctx->impl;
        c->activate();
        Scene s(c, *g);
        Batch b(c);
        b.prepare(s, {*cam});
        *n_entries = b.n_entries;
        SLM_CUDA_CHECK(cudaMemcpyAsync(offsets, b.tile_offsets.p, sizeof(int) * (b.n_tiles + 1), cudaMemcpyDeviceToHost, c->stream));
        if (b.n_entries <= capacity)
            SLM_CUDA_CHECK(cudaMemcpyAsync(indices, b.entries.p, sizeof(int) * b.n_entries, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    });
}

int slm_prepare(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam, double* mean2d, double* conic,
                double* opacity, double* color, double* depth, double* radius, int32_t* valid) {
    return guarded([&] {
        Context* c = &ctx->impl;
        c->activate();
        Scene s(c, *g);
        Batch b(c);
        b.prepare(s, {*cam});
        const int G = s.G;
        std::vector<float4> rec(3 * static_cast<size_t>(s.Gp));
        std::vector<unsigned long long> keys(s.Gp);
        SLM_CUDA_CHECK(cudaMemcpyAsync(rec.data(), b.rec.p, sizeof(float4) * rec.size(), cudaMemcpyDeviceToHost, c->stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(keys.data(), b.keys.p, sizeof(unsigned long long) * keys.size(), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        const double ln2 = 0.69314718055994530942;
        for (int i = 0; i < G; ++i) {
            const float4 r0 = rec[3 * i], r1 = rec[3 * i + 1], r2 = rec[3 * i + 2];
            valid[i] = r2.y != 0.f;
            mean2d[2 * i] = r0.x;
            mean2d[2 * i + 1] = r0.y;
            conic[3 * i] = -2.0 * ln2 * r0.z;
            conic[3 * i + 1] = -ln2 * r0.w;
            conic[3 * i + 2] = -2.0 * ln2 * r1.x;
            opacity[i] = r1.y;
            color[3 * i] = r1.z;
            color[3 * i + 1] = r1.w;
            color[3 * i + 2] = r2.x;
            unsigned long long k = keys[i];
            k = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
            double d;
            std::memcpy(&d, &k, sizeof d);
            depth[i] = d;
            radius[i] = 0.0;
        }
    });
}

int slm_render_full(slm_context* ctx, const slm_gaussians* g, const slm_camera* cam, double* image,
                    double* transmittance, int32_t* contrib) {
    return guarded([&] {
        Context* c = &ctx->impl;
        c->activate();
        Scene s(c, *g);
        Batch b(c);
        b.prepare(s, {*cam});
        // the reference's blend replayed in FP64 (k_render_exact): contrib / T are
        // its decisions, the image its values up to FP32-stored colours
        const size_t np = static_cast<size_t>(cam->width) * cam->height;
        DevBuf<double> dimg, dtr;
        DevBuf<int> dcn;
        dimg.ensure(std::max<size_t>(3 * np, 1));
        dtr.ensure(std::max<size_t>(np, 1));
        dcn.ensure(std::max<size_t>(np, 1));
        launch_render_exact(b.cams.p, b.tile_view.p, b.n_tiles, b.tile_offsets.p, b.entries.p, b.rec64.p, b.rec.p, b.Gp,
                            dimg.p, dtr.p, dcn.p, c->stream);
        c->check_launch();
        if (image) SLM_CUDA_CHECK(cudaMemcpyAsync(image, dimg.p, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost, c->stream));
        if (transmittance)
            SLM_CUDA_CHECK(cudaMemcpyAsync(transmittance, dtr.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c->stream));
        if (contrib) SLM_CUDA_CHECK(cudaMemcpyAsync(contrib, dcn.p, sizeof(int) * np, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    });
}

int slm_render_pixel(slm_context* ctx, int n, const double* splats, double px, double py, double out[4],
                     int32_t* contrib) {
    return guarded([&] {  // render::render_pixel (rasterizer.cpp:52-60)
        if (n < 0) throw std::invalid_argument("render_pixel: negative splat count");
        Context& c = ctx->impl;
        c.activate();
        DevBuf<double> d, o;
        DevBuf<int> cn;
        d.ensure(static_cast<size_t>(std::max(n, 1)) * 10);
        o.ensure(4);
        cn.ensure(1);
        if (n) SLM_CUDA_CHECK(cudaMemcpyAsync(d.p, splats, sizeof(double) * 10 * n, cudaMemcpyHostToDevice, c.stream));
        launch_render_pixel(n, d.p, px, py, o.p, cn.p, c.stream);
        c.check_launch();
        SLM_CUDA_CHECK(cudaMemcpyAsync(out, o.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(contrib, cn.p, sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}
int slm_render_splats(slm_context* ctx, const slm_camera* cam, int n_splats, const double* splats,
                      const int32_t* offsets, const int32_t* indices, double* image, double* transmittance,
                      int32_t* contrib) {
    return guarded([&] {  // render::render_with_context (rasterizer.cpp:62-91)
        if (cam->width <= 0 || cam->height <= 0) throw std::invalid_argument("camera size must be positive");
        Context& c = ctx->impl;
        c.activate();
        const int tx = (cam->width + kTile - 1) / kTile, ty = (cam->height + kTile - 1) / kTile, nt = tx * ty;
        const long long ne = offsets[nt];
        for (int t = 0; t < nt; ++t)
            if (offsets[t] > offsets[t + 1]) throw std::invalid_argument("render_with_context: bad tile offsets");
        for (long long k = 0; k < ne; ++k)
            if (indices[k] < 0 || indices[k] >= n_splats) throw std::invalid_argument("render_with_context: index");
        DevBuf<double> d, img, tr;
        DevBuf<int> off, lst, cn;
        const size_t np = static_cast<size_t>(cam->width) * cam->height;
        d.ensure(static_cast<size_t>(std::max(n_splats, 1)) * 10);
        off.ensure(nt + 1);
        lst.ensure(std::max<long long>(ne, 1));
        img.ensure(3 * np);
        tr.ensure(np);
        cn.ensure(np);
        if (n_splats)
            SLM_CUDA_CHECK(cudaMemcpyAsync(d.p, splats, sizeof(double) * 10 * n_splats, cudaMemcpyHostToDevice, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(off.p, offsets, sizeof(int) * (nt + 1), cudaMemcpyHostToDevice, c.stream));
        if (ne) SLM_CUDA_CHECK(cudaMemcpyAsync(lst.p, indices, sizeof(int) * ne, cudaMemcpyHostToDevice, c.stream));
        launch_render_splats(cam->width, cam->height, tx, nt, off.p, lst.p, d.p, img.p, tr.p, cn.p, c.stream);
        c.check_launch();
        SLM_CUDA_CHECK(cudaMemcpyAsync(image, img.p, sizeof(double) * 3 * np, cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(transmittance, tr.p, sizeof(double) * np, cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(contrib, cn.p, sizeof(int) * np, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}
int slm_residuals(const double* rendered, const double* truth, int64_t n, double* out) {
    return guarded([&] {  // render::residuals (rasterizer.cpp:97-104): elementwise rendered - truth (host)
        if (n < 0) throw std::invalid_argument("residuals: negative length");
        for (int64_t i = 0; i < n; ++i) out[i] = rendered[i] - truth[i];
    });
}
int slm_debug_nccl_selftest(slm_context* ctx, double* out) {
    return guarded([&] {
        Context& c = ctx->impl;
        c.activate();
        ncclUniqueId uid;
        SLM_NCCL_CHECK(nccl().GetUniqueId(&uid));
        NcclComm nc;
        SLM_NCCL_CHECK(nccl().CommInitRank(&nc.c, 1, uid, 0));
        const size_t n = 4 * 1000 + 7, pitch = 1024, rows = 4, len = 1000;
        std::vector<float> hf(n);
        std::vector<double> hd(n);
        for (size_t i = 0; i < n; ++i) {
            hf[i] = static_cast<float>(i) * 0.25f - 3.0f;
            hd[i] = static_cast<double>(i) * 0.125 + 1.0;
        }
        DevBuf<float> df;
        DevBuf<double> dd;
        df.ensure(n);
        dd.ensure(n);
        SLM_CUDA_CHECK(cudaMemcpyAsync(df.p, hf.data(), n * sizeof(float), cudaMemcpyHostToDevice, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(dd.p, hd.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        nc.allreduce(df.p, n, false, c.stream);
        nc.allreduce(dd.p, n, true, c.stream);
        nc.allreduce_rows(df.p, pitch, static_cast<int>(rows), len, c.stream);
        std::vector<float> rf(n);
        std::vector<double> rd(n);
        SLM_CUDA_CHECK(cudaMemcpyAsync(rf.data(), df.p, n * sizeof(float), cudaMemcpyDeviceToHost, c.stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(rd.data(), dd.p, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        double err = 0.0;
        for (size_t i = 0; i < n; ++i) {
            err = std::max(err, std::fabs(static_cast<double>(rf[i]) - hf[i]));
            err = std::max(err, std::fabs(rd[i] - hd[i]));
        }
        out[0] = err;
        out[1] = static_cast<double>(2 * n);
    });
}
int slm_debug_render_stats(slm_scene* s, const slm_camera* cams, int n_cams, uint64_t* out) {
    return guarded([&] {  // k_render work counters: [entry iterations (per thread), past the box test,
                          //  live pixel-entry gate evaluations, blends, staged entries (per thread)]
        Context* c = s->impl.ctx;
        c->activate();
        Batch b(c);
        b.prepare(s->impl, std::vector<slm_camera>(cams, cams + n_cams));
        b.image.ensure(3 * std::max<long long>(b.n_pix, 1));
        b.trans.ensure(std::max<long long>(b.n_pix, 1));
        b.contrib.ensure(std::max<long long>(b.n_pix, 1));
        b.last.ensure(std::max<long long>(b.n_pix, 1));
        DevBuf<unsigned long long> d;
        d.ensure(10);
        SLM_CUDA_CHECK(cudaMemsetAsync(d.p, 0, 10 * sizeof(unsigned long long), c->stream));
        launch_render(b.cams.p, b.tile_view.p, b.n_tiles, b.tile_offsets.p, b.entries.p, b.rec.p, b.Gp, nullptr,
                      b.image.p, b.trans.p, b.contrib.p, b.last.p, nullptr, c->stream, d.p);
        SLM_CUDA_CHECK(cudaMemcpyAsync(out, d.p, 5 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        // [8] warps past the exact ellipse/half-tile test, [9] warp-entries where some pixel blended
        SLM_CUDA_CHECK(cudaMemcpyAsync(out + 8, d.p + 8, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        out[5] = static_cast<uint64_t>(b.n_entries);
        out[6] = static_cast<uint64_t>(b.n_pix);
        out[7] = static_cast<uint64_t>(b.n_tiles);
    });
}
int slm_scene_render(slm_scene* s, const slm_camera* cam, float* image, float* transmittance, int32_t* contrib) {
    return guarded([&] {
        Context* c = s->impl.ctx;
        c->activate();
        Batch b(c);
        b.prepare(s->impl, {*cam});
        b.render(false);
        const size_t np = static_cast<size_t>(cam->width) * cam->height;
        if (image) SLM_CUDA_CHECK(cudaMemcpyAsync(image, b.image.p, sizeof(float) * 3 * np, cudaMemcpyDeviceToHost, c->stream));
        if (transmittance) SLM_CUDA_CHECK(cudaMemcpyAsync(transmittance, b.trans.p, sizeof(float) * np, cudaMemcpyDeviceToHost, c->stream));
        if (contrib) SLM_CUDA_CHECK(cudaMemcpyAsync(contrib, b.contrib.p, sizeof(int) * np, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    });
}

int slm_build_sample_plan(const slm_camera* cams, int n_cams, int samples_per_tile, int dist, int lane_width,
                          slm_rng* rng, const double* const* aux_image, const int32_t* const* aux_contrib,
                          const double* const* aux_gt, slm_plan_h** out) {
    return guarded([&] {
        auto p = build_plan(cams, n_cams, samples_per_tile, dist, lane_width, rng->eng, aux_image, aux_contrib, aux_gt);
        *out = new slm_plan_h{std::move(p)};
    });
}
int slm_exhaustive_plan(const slm_camera* cams, int n_cams, slm_plan_h** out) {
    return guarded([&] { *out = new slm_plan_h{exhaustive(cams, n_cams)}; });
}
void slm_plan_destroy(slm_plan_h* p) { delete p; }
int slm_plan_size(slm_plan_h* p, int* n_views, int64_t* total) {
    *n_views = static_cast<int>(p->impl->view_camera.size());
    *total = p->impl->view_offset.back();
    return SLM_OK;
}
int slm_plan_export(slm_plan_h* p, int32_t* view_camera, int64_t* view_offset, int32_t* px, int32_t* py,
                    int32_t* tile, double* weight) {
    const PlanH& h = *p->impl;
    std::copy(h.view_camera.begin(), h.view_camera.end(), view_camera);
    std::copy(h.view_offset.begin(), h.view_offset.end(), view_offset);
    std::copy(h.px.begin(), h.px.end(), px);
    std::copy(h.py.begin(), h.py.end(), py);
    std::copy(h.tile.begin(), h.tile.end(), tile);
    std::copy(h.weight.begin(), h.weight.end(), weight);
    return SLM_OK;
}
int slm_estimate_loss(const slm_camera* cams, const slm_plan* plan, const double* const* fields, double* out) {
    return guarded([&] {  // sample_plan.cpp:199-222 (host: O(samples) gather, not on the hot path)
        const long long n_total = plan->view_offset[plan->n_views];
        if (n_total == 0) {
            *out = 0.0;
            return;
        }
        double pixels = 0.0;
        for (int v = 0; v < plan->n_views; ++v) {
            if (!fields || !fields[v]) throw std::invalid_argument("one residual field per plan view required");
            pixels += static_cast<double>(cams[plan->view_camera[v]].width) * cams[plan->view_camera[v]].height;
        }
        double acc = 0.0;
        for (int v = 0; v < plan->n_views; ++v) {
            const int w = cams[plan->view_camera[v]].width;
            for (long long s = plan->view_offset[v]; s < plan->view_offset[v + 1]; ++s) {
                double sq = 0.0;
                for (int c = 0; c < 3; ++c) {
                    const double r = fields[v][(static_cast<size_t>(plan->py[s]) * w + plan->px[s]) * 3 + c];
                    sq += r * r;
                }
                acc += plan->weight[s] * sq;
            }
        }
        *out = acc / (static_cast<double>(n_total) * pixels * 3.0);
    });
}
int slm_camera_features(const slm_camera* cams, int n_cams, double* feats) {
    return guarded([&] {
        const auto f = features(cams, n_cams);
        for (int i = 0; i < n_cams; ++i)
            for (int d = 0; d < 6; ++d) feats[6 * i + d] = f[i][d];
    });
}
int slm_kmeans_cameras(const slm_camera* cams, int n_cams, int k, uint64_t seed, int32_t* assign) {
    return guarded([&] {
        const auto a = kmeans(features(cams, n_cams), k, seed);
        std::copy(a.begin(), a.end(), assign);
    });
}
int slm_sample_view_batch(const int32_t* assign, int n_cams, int k, slm_rng* rng, int32_t* batch) {
    return guarded([&] {
        const auto b = view_batch(std::vector<int>(assign, assign + n_cams), k, rng->eng);
        std::copy(b.begin(), b.end(), batch);
    });
}

int slm_jacobian_create(slm_context* ctx, const slm_gaussians* g, const slm_camera* cams, int n_cams,
                        const slm_plan* plan, slm_jacobian** out) {
    *out = nullptr;
    return guarded([&] {
        Context* c = &ctx->impl;
        c->activate();
        auto h = std::make_unique<slm_jacobian>();
        h->scene = std::make_unique<Scene>(c, *g);  // SampledJacobian copies the set (jacobian.cpp:100)
        make_jacobian(c, h->scene.get(), cams, n_cams, *plan, h.get());
        *out = h.release();
    });
}
int slm_jacobian_create_scene(slm_scene* s, const slm_camera* cams, int n_cams, const slm_plan* plan,
                              slm_jacobian** out) {
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<slm_jacobian>();
        make_jacobian(s->impl.ctx, &s->impl, cams, n_cams, *plan, h.get());
        *out = h.release();
    });
}
void slm_jacobian_destroy(slm_jacobian* j) { delete j; }
int slm_jacobian_dims(slm_jacobian* j, int64_t* rdim, int64_t* pdim) {
    *rdim = j->jac->rdim;
    *pdim = static_cast<int64_t>(kP) * j->jac->scene->G;
    return SLM_OK;
}
int slm_jacobian_jvp(slm_jacobian* j, const double* v, double* out) {
    return guarded([&] { j->jac->ctx->activate(); j->jac->jvp(v, out); });
}
int slm_jacobian_vjp(slm_jacobian* j, const double* u, double* out) {
    return guarded([&] { j->jac->ctx->activate(); j->jac->vjp(u, out); });
}
int slm_jacobian_jtj_diag(slm_jacobian* j, double* out) {
    return guarded([&] { j->jac->ctx->activate(); j->jac->jtj_diag(out); });
}
int slm_jacobian_gn_apply(slm_jacobian* j, double lambda, const double* p, double* out) {
    return guarded([&] { j->jac->ctx->activate(); j->jac->gn_apply(lambda, p, out); });
}
int slm_jacobian_weights(slm_jacobian* j, double* out) {
    return guarded([&] {
        const auto& w = j->jac->residual_weights();
        std::copy(w.begin(), w.end(), out);
    });
}
int slm_jacobian_set_weights(slm_jacobian* j, const double* w) {
    return guarded([&] {
        Jacobian& J = *j->jac;
        J.weights.assign(w, w + J.rdim);
        J.samples.upload_weights(J.ctx, J.weights);
    });
}
int slm_jacobian_gn_apply_dev(slm_jacobian* j, float lambda, const float* d_p, float* d_out) {
    return guarded([&] { j->jac->gn_apply_dev(lambda, d_p, d_out); });
}
int slm_jacobian_device_ptrs(slm_jacobian* j, void* stream_out[1]) {
    stream_out[0] = j->jac->ctx->stream;
    return SLM_OK;
}
int slm_jacobian_stats(slm_jacobian* j, int64_t* out) {
    // [views, sum_v G_v, entries, samples, groups, tiles]
    Batch& b = *j->jac->batch;
    out[0] = b.V;
    out[1] = std::accumulate(b.valid_count.begin(), b.valid_count.end(), 0ll);
    out[2] = b.n_entries;
    out[3] = j->jac->samples.total;
    out[4] = static_cast<int64_t>(j->jac->samples.hgroups.size());
    out[5] = b.n_tiles;
    return SLM_OK;
}
int slm_jacobian_mask_stats(slm_jacobian* j, uint64_t* out) {
    return guarded([&] {
        Jacobian& J = *j->jac;
        J.ctx->activate();
        DevBuf<unsigned long long> d;
        d.ensure(18);
        SLM_CUDA_CHECK(cudaMemsetAsync(d.p, 0, 18 * sizeof(unsigned long long), J.ctx->stream));
        launch_mask_stats(J.args(), d.p, J.ctx->stream);
        SLM_CUDA_CHECK(cudaMemcpyAsync(out, d.p, 18 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, J.ctx->stream));
        J.ctx->sync();
    });
}
int slm_jacobian_pcg(slm_jacobian* j, double lambda, const double* b, const double* minv, int max_iters,
                     double* x, slm_pcg_result* res) {
    return guarded([&] {
        Jacobian& J = *j->jac;
        J.ctx->activate();
        DevBuf<float> db, dm, dx;
        db.ensure(J.P());
        dm.ensure(J.P());
        dx.ensure(J.P());
        J.upload_param(b, db.p);
        J.upload_param(minv, dm.p);
        const CgState cs = J.pcg_dev(static_cast<float>(lambda), db.p, dm.p, max_iters, dx.p);
        J.download_param(dx.p, x);
        res->iterations = cs.iterations;
        res->breakdown = cs.breakdown;
        res->rel_residual = cs.bnorm == 0.0 ? 0.0 : std::sqrt(cs.rr) / cs.bnorm;
    });
}

int slm_pcg_solve(slm_context* ctx, slm_apply_fn apply, void* user, const double* b, const double* minv,
                  int64_t n, int max_iters, double* x, slm_pcg_result* res) {
    return guarded([&] {
        // Vector algebra on the device (f32 storage, f64 reductions); the
        // caller's operator runs on host vectors between the device steps.
        Context& c = ctx->impl;
        c.activate();
        const long long np = (n + 3) / 4 * 4;
        DevBuf<float> db, dm, dx, dr, dz, dp, du;
        for (auto* buf : {&db, &dm, &dx, &dr, &dz, &dp, &du}) {
            buf->ensure(np);
            SLM_CUDA_CHECK(cudaMemsetAsync(buf->p, 0, np * sizeof(float), c.stream));
        }
        std::vector<float> hf(n);
        std::vector<double> hp(n), hu(n);
        auto up = [&](const double* src, float* dst) {
            for (int64_t i = 0; i < n; ++i) hf[i] = static_cast<float>(src[i]);
            SLM_CUDA_CHECK(cudaMemcpyAsync(dst, hf.data(), sizeof(float) * n, cudaMemcpyHostToDevice, c.stream));
            c.sync();
        };
        auto down = [&](const float* src, double* dst) {
            SLM_CUDA_CHECK(cudaMemcpyAsync(hf.data(), src, sizeof(float) * n, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int64_t i = 0; i < n; ++i) dst[i] = hf[i];
        };
        up(b, db.p);
        up(minv, dm.p);
        CgState* cg = c.cg.p;
        launch_cg_init(db.p, dm.p, np, dx.p, dr.p, dz.p, dp.p, c.partial.p, cg, c.stream);
        CgState h;
        for (int it = 0; it < max_iters; ++it) {
            SLM_CUDA_CHECK(cudaMemcpyAsync(&h, cg, sizeof h, cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            if (h.done) break;
            down(dp.p, hp.data());
            apply(user, hp.data(), hu.data());
            up(hu.data(), du.p);
            launch_cg_pu(dp.p, du.p, np, c.partial.p, cg, c.stream);
            launch_cg_update(dx.p, dr.p, dz.p, dp.p, du.p, dm.p, np, c.partial.p, cg, c.stream);
        }
        c.check_launch();
        SLM_CUDA_CHECK(cudaMemcpyAsync(&h, cg, sizeof h, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        down(dx.p, x);
        res->iterations = h.iterations;
        res->breakdown = h.breakdown;
        res->rel_residual = h.bnorm == 0.0 ? 0.0 : std::sqrt(h.rr) / h.bnorm;
    });
}

void slm_default_lm_config(slm_lm_config* c) {
    *c = slm_lm_config{0.1, 3, 8, 50, 8, 8, 50, 32, 32, 0.2, 0.05, 10, SLM_DIST_UNIFORM, SLM_LOSS_MSE, 0.2};
}

int slm_learning_rate(slm_context* ctx, const double* delta, int64_t n, int iteration, const slm_lm_config* cfg,
                      double* eta) {
    return guarded([&] {
        if (n % kP != 0) throw std::invalid_argument("learning_rate: bad update length");
        Context& c = ctx->impl;
        c.activate();
        const int G = static_cast<int>(n / kP);
        const int Gp = round_up(std::max(G, 1), 256);
        DevBuf<double> a;
        DevBuf<float> s, m;
        a.ensure(std::max<int64_t>(n, 1));
        s.ensure(static_cast<size_t>(kP) * Gp);
        m.ensure(1);
        SLM_CUDA_CHECK(cudaMemcpyAsync(a.p, delta, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
        launch_aos64_to_soa32(a.p, G, Gp, s.p, c.stream);
        launch_color_maxabs(s.p, G, Gp, m.p, c.stream);
        float hm = 0.f;
        SLM_CUDA_CHECK(cudaMemcpyAsync(&hm, m.p, sizeof(float), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        *eta = learning_rate_from(hm, iteration, *cfg);
    });
}

int slm_train_create(slm_context* ctx, const slm_camera* cams, int n_cams, const float* images, slm_train** out) {
    return guarded([&] {
        Context* c = &ctx->impl;
        c->activate();
        auto t = std::make_unique<slm_train>();
        t->impl.ctx = c;
        t->impl.cams.assign(cams, cams + n_cams);
        size_t off = 0;
        for (int i = 0; i < n_cams; ++i) {
            t->impl.img_off.push_back(off);
            off += 3 * static_cast<size_t>(cams[i].width) * cams[i].height;
        }
        t->impl.images.ensure(std::max<size_t>(off, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(t->impl.images.p, images, sizeof(float) * off, cudaMemcpyHostToDevice, c->stream));
        c->sync();
        *out = t.release();
    });
}
void slm_train_destroy(slm_train* t) { delete t; }
int slm_train_rebuild_clusters(slm_train* t, int k, uint64_t seed) {
    return guarded([&] {
        auto& T = t->impl;
        T.assign = kmeans(features(T.cams.data(), static_cast<int>(T.cams.size())), k, seed);
        T.k = k;
    });
}
int slm_train_set_clusters(slm_train* t, const int32_t* assign, int k) {
    return guarded([&] {
        t->impl.assign.assign(assign, assign + t->impl.cams.size());
        t->impl.k = k;
    });
}
int slm_train_clusters(slm_train* t, int32_t* assign, int* k) {
    std::copy(t->impl.assign.begin(), t->impl.assign.end(), assign);
    *k = t->impl.k;
    return SLM_OK;
}

int slm_lm_step(slm_scene* s, slm_train* t, const slm_lm_config* cfg, int iteration, slm_rng* rng,
                slm_step_report* report) {
    return guarded([&] { lm_step(s->impl, t->impl, *cfg, iteration, rng->eng, *report); });
}

int slm_lm_step_host(slm_context* ctx, slm_gaussians* state, slm_train* t, const slm_lm_config* cfg,
                     int iteration, slm_rng* rng, slm_step_report* report) {
    return guarded([&] {
        Scene s(&ctx->impl, *state);
        lm_step(s, t->impl, *cfg, iteration, rng->eng, *report);
        s.download(*state);
    });
}

int slm_batch_loss(slm_scene* s, slm_train* t, const int32_t* cam_ids, int n, double* out) {
    return slm_batch_loss_kind(s, t, cam_ids, n, SLM_LOSS_MSE, 0.0, out);
}

int slm_batch_loss_kind(slm_scene* s, slm_train* t, const int32_t* cam_ids, int n, int loss, double ssim_weight,
                        double* out) {
    return guarded([&] {
        Context* c = s->impl.ctx;
        c->activate();
        Batch b(c);
        *out = batch_loss_dev(s->impl, t->impl, std::vector<int>(cam_ids, cam_ids + n), loss, ssim_weight, b);
    });
}

// ---- first-order baselines (baselines/first_order.hpp) on the device
struct slm_first_order {
    FirstOrder impl;  // built in place: its Jacobian points at its own Batch
    explicit slm_first_order(Scene* s) : impl(s) {}
};

void slm_default_first_order_config(slm_first_order_config* c) {
    *c = slm_first_order_config{SLM_FO_ADAM, 1.6e-3, 2.5e-2, 5e-2, 5e-3, 1e-3, 0.9, 0.999, 1e-15, 0.99, 1e-15,
                                0.99, 0.01, 0, SLM_LOSS_MSE, 0.2};
}

int slm_full_gradient(slm_scene* s, slm_train* t, int loss, double ssim_weight, double* grad_aos) {
    return guarded([&] {
        Context* c = s->impl.ctx;
        c->activate();
        Batch b(c);
        Jacobian j(c, &s->impl, &b);
        DevBuf<float> grad, chunk;
        grad.ensure(s->impl.P());
        full_gradient_dev(s->impl, t->impl, loss, ssim_weight, b, j, chunk, grad.p);
        DevBuf<double> stage;
        stage.ensure(std::max<size_t>(static_cast<size_t>(kP) * s->impl.G, 1));
        launch_soa32_to_aos64(grad.p, s->impl.G, s->impl.Gp, stage.p, c->stream);
        c->check_launch();
        SLM_CUDA_CHECK(cudaMemcpyAsync(grad_aos, stage.p, sizeof(double) * kP * s->impl.G, cudaMemcpyDeviceToHost,
                                       c->stream));
        c->sync();
    });
}

int slm_first_order_create(slm_scene* s, slm_first_order** out) {
    return guarded([&] {
        s->impl.ctx->activate();
        *out = new slm_first_order(&s->impl);
    });
}

void slm_first_order_destroy(slm_first_order* f) {
    if (f) {
        f->impl.scene->ctx->activate();
        delete f;
    }
}

static void soa64_to_aos(const FirstOrder& f, const DevBuf<double>& m, double* out) {
    const int G = f.scene->G, Gp = f.scene->Gp;
    std::vector<double> h(static_cast<size_t>(kP) * Gp);
    SLM_CUDA_CHECK(cudaMemcpyAsync(h.data(), m.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, f.scene->ctx->stream));
    f.scene->ctx->sync();
    for (int g = 0; g < G; ++g)
        for (int k = 0; k < kP; ++k) out[static_cast<size_t>(g) * kP + k] = h[static_cast<size_t>(k) * Gp + g];
}

static void aos_to_soa64(FirstOrder& f, const double* in, DevBuf<double>& m) {
    const int G = f.scene->G, Gp = f.scene->Gp;
    std::vector<double> h(static_cast<size_t>(kP) * Gp, 0.0);
    for (int g = 0; g < G; ++g)
        for (int k = 0; k < kP; ++k) h[static_cast<size_t>(k) * Gp + g] = in[static_cast<size_t>(g) * kP + k];
    SLM_CUDA_CHECK(cudaMemcpyAsync(m.p, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, f.scene->ctx->stream));
    f.scene->ctx->sync();
}

int slm_first_order_moments(slm_first_order* f, double* m1, double* m2, int64_t* step) {
    return guarded([&] {
        f->impl.scene->ctx->activate();
        if (m1) soa64_to_aos(f->impl, f->impl.m1, m1);
        if (m2) soa64_to_aos(f->impl, f->impl.m2, m2);
        if (step) *step = f->impl.step;
    });
}

int slm_first_order_set_moments(slm_first_order* f, const double* m1, const double* m2, int64_t step) {
    return guarded([&] {
        f->impl.scene->ctx->activate();
        if (step < 0) throw std::invalid_argument("first-order step must be non-negative");
        aos_to_soa64(f->impl, m1, f->impl.m1);
        aos_to_soa64(f->impl, m2, f->impl.m2);
        f->impl.step = step;
    });
}

int slm_first_order_apply(slm_first_order* f, const double* grad_aos, const slm_first_order_config* cfg) {
    return guarded([&] {
        FirstOrder& F = f->impl;
        Context* c = F.scene->ctx;
        c->activate();
        const size_t n = static_cast<size_t>(kP) * F.scene->G;
        F.g64.ensure(std::max<size_t>(n, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(F.g64.p, grad_aos, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        F.apply(nullptr, F.g64.p, *cfg);
        c->sync();
    });
}

int slm_first_order_step(slm_first_order* f, slm_train* t, const slm_first_order_config* cfg, double* train_loss) {
    return guarded([&] {  // one train_run iteration of a first-order optimizer (run.cpp:176-182)
        FirstOrder& F = f->impl;
        Context* c = F.scene->ctx;
        c->activate();
        F.grad.ensure(F.scene->P());
        full_gradient_dev(*F.scene, t->impl, cfg->loss, cfg->ssim_weight, F.batch, F.jac, F.chunk, F.grad.p);
        F.apply(F.grad.p, nullptr, *cfg);
        if (train_loss) {
            std::vector<int> ids(t->impl.cams.size());
            std::iota(ids.begin(), ids.end(), 0);
            *train_loss = batch_loss_dev(*F.scene, t->impl, ids, cfg->loss, cfg->ssim_weight, F.batch);
        }
        c->sync();
    });
}

int slm_evaluate(slm_context* ctx, const double* rendered, const double* gt, int width, int height,
                 slm_metric_report* out) {
    return guarded([&] {
        if (width < 0 || height < 0) throw std::invalid_argument("metrics: image shapes differ");
        Context* c = &ctx->impl;
        c->activate();
        const size_t n = 3 * static_cast<size_t>(width) * height;
        DevBuf<double> da, db;
        da.ensure(std::max<size_t>(n, 1));
        db.ensure(std::max<size_t>(n, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(da.p, rendered, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(db.p, gt, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        const auto s = image_metrics<double>(c, da.p, db.p, {ImageRef{0, width, height}});
        *out = metric_report(s[0], width, height);
    });
}

int slm_ssim_diag_residuals(slm_context* ctx, const double* a, const double* b, int width, int height,
                            double* residual, double* d_center) {
    return guarded([&] {
        if (width < 0 || height < 0) throw std::invalid_argument("metrics: image shapes differ");
        Context* c = &ctx->impl;
        c->activate();
        const size_t n = 3 * static_cast<size_t>(width) * height;
        DevBuf<double> da, db, dr, dd;
        for (DevBuf<double>* p : {&da, &db, &dr, &dd}) p->ensure(std::max<size_t>(n, 1));
        SLM_CUDA_CHECK(cudaMemcpyAsync(da.p, a, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(db.p, b, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        image_metrics<double>(c, da.p, db.p, {ImageRef{0, width, height}}, true, dr.p, dd.p);
        SLM_CUDA_CHECK(cudaMemcpyAsync(residual, dr.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        SLM_CUDA_CHECK(cudaMemcpyAsync(d_center, dd.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
    });
}

int slm_evaluate_split(slm_scene* s, slm_train* split, slm_metric_report* out) {
    return guarded([&] {  // io::evaluate_split (run.cpp:77-92): render_full + evaluate per camera, mean
        Context* c = s->impl.ctx;
        c->activate();
        Train& t = split->impl;
        const int n = static_cast<int>(t.cams.size());
        slm_metric_report mean{};
        constexpr int kChunk = 8;  // views rendered per batch (bounds the batch buffers)
        for (int lo = 0; lo < n; lo += kChunk) {
            const int hi = std::min(n, lo + kChunk);
            std::vector<int> ids;
            std::vector<slm_camera> cv;
            for (int i = lo; i < hi; ++i) {
                ids.push_back(i);
                cv.push_back(t.cams[i]);
            }
            Batch b(c);
            b.prepare(s->impl, cv);
            copy_gt(t, b, ids);
            b.render(false, false);
            std::vector<ImageRef> imgs;
            for (int v = 0; v < b.V; ++v) imgs.push_back({3 * b.hcams[v].pix_base, cv[v].width, cv[v].height});
            const auto sums = image_metrics<float>(c, b.image.p, b.gt.p, imgs);
            for (int v = 0; v < b.V; ++v) {
                const slm_metric_report r = metric_report(sums[v], cv[v].width, cv[v].height);
                mean.mse += r.mse;
                mean.psnr += r.psnr;
                mean.ssim += r.ssim;
            }
        }
        if (n > 0) {
            mean.mse /= n;
            mean.psnr /= n;
            mean.ssim /= n;
        }
        *out = mean;
    });
}

// ---- checkpoints (io/checkpoint.cpp:12-82): "SPLMGS01", u32 version 1,
// u64 count, then the ParamVector as little-endian f64 (14 per Gaussian), plus
// the .meta.txt sidecar -- byte-identical to the reference's files.
namespace {
constexpr char kCkptMagic[8] = {'S', 'P', 'L', 'M', 'G', 'S', '0', '1'};
constexpr uint32_t kCkptVersion = 1;

void put_le(std::ostream& out, uint64_t v, int bytes) {
    char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
    out.write(b, bytes);
}
uint64_t get_le(std::istream& in, int bytes) {
    unsigned char b[8] = {};
    in.read(reinterpret_cast<char*>(b), bytes);
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return v;
}
void pack_set(const slm_gaussians& g, std::vector<double>& p) {  // GaussianSet::pack (types.cpp:20-33)
    p.resize(static_cast<size_t>(kP) * g.count);
    for (int i = 0; i < g.count; ++i) {
        double* b = p.data() + static_cast<size_t>(kP) * i;
        for (int k = 0; k < 3; ++k) b[k] = g.means[3 * i + k];
        for (int k = 0; k < 3; ++k) b[3 + k] = g.log_scales[3 * i + k];
        for (int k = 0; k < 4; ++k) b[6 + k] = g.rotations[4 * i + k];
        b[10] = g.opacity_logits[i];
        for (int k = 0; k < 3; ++k) b[11 + k] = g.colors[3 * i + k];
    }
}
// reads the header; returns the Gaussian count (stream positioned at the parameters)
uint64_t read_header(std::ifstream& in, const std::string& path) {
    char magic[8];
    in.read(magic, 8);
    if (!in || std::memcmp(magic, kCkptMagic, 8) != 0) throw std::runtime_error("not a splatlm checkpoint: " + path);
    if (get_le(in, 4) != kCkptVersion) throw std::runtime_error("unsupported checkpoint version in " + path);
    return get_le(in, 8);
}
}  // namespace

int slm_save_checkpoint(const char* path, const slm_gaussians* g) {
    return guarded([&] {
        std::ofstream out(path, std::ios::binary);
        if (!out) throw std::runtime_error(std::string("cannot write checkpoint: ") + path);
        out.write(kCkptMagic, sizeof kCkptMagic);
        put_le(out, kCkptVersion, 4);
        put_le(out, static_cast<uint64_t>(g->count), 8);
        std::vector<double> p;
        pack_set(*g, p);
        for (double d : p) {
            uint64_t u;
            std::memcpy(&u, &d, 8);
            put_le(out, u, 8);
        }
        if (!out) throw std::runtime_error(std::string("checkpoint write failed: ") + path);
        std::ofstream meta(std::string(path) + ".meta.txt");
        meta << "splatlm checkpoint v" << kCkptVersion << "\n"
             << "gaussians: " << g->count << "\n"
             << "parameters: " << p.size() << "\n"
             << "layout: per-Gaussian [mean(3), log_scale(3), rotation wxyz(4), "
                "opacity_logit(1), color(3)], little-endian float64\n";
    });
}

int slm_checkpoint_count(const char* path, int* count) {
    return guarded([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot read checkpoint: ") + path);
        *count = static_cast<int>(read_header(in, path));
    });
}

int slm_load_checkpoint(const char* path, slm_gaussians* out) {
    return guarded([&] {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot read checkpoint: ") + path);
        const uint64_t count = read_header(in, path);
        if (static_cast<int64_t>(count) != out->count)
            throw std::invalid_argument("load_checkpoint: output GaussianSet has the wrong count");
        std::vector<double> p(static_cast<size_t>(kP) * count);
        for (double& d : p) {
            const uint64_t u = get_le(in, 8);
            std::memcpy(&d, &u, 8);
        }
        if (!in) throw std::runtime_error(std::string("truncated checkpoint: ") + path);
        for (uint64_t i = 0; i < count; ++i) {  // GaussianSet::unpack (types.cpp:35-46)
            const double* b = p.data() + kP * i;
            for (int k = 0; k < 3; ++k) out->means[3 * i + k] = b[k];
            for (int k = 0; k < 3; ++k) out->log_scales[3 * i + k] = b[3 + k];
            for (int k = 0; k < 4; ++k) out->rotations[4 * i + k] = b[6 + k];
            out->opacity_logits[i] = b[10];
            for (int k = 0; k < 3; ++k) out->colors[3 * i + k] = b[11 + k];
        }
    });
}

int slm_random_init(int count, const double* lo, const double* hi, slm_rng* rng, slm_gaussians* out) {
    return guarded([&] {  // io::random_init (dataset.cpp:138-166)
        if (count < 1) throw std::invalid_argument("random_init: count must be at least 1");
        std::uniform_real_distribution<double> ux(lo[0], hi[0]), uy(lo[1], hi[1]), uz(lo[2], hi[2]);
        const double coeff_max = 0.5 / 0.28209479177387814;
        std::uniform_real_distribution<double> ucolor(-coeff_max, coeff_max);
        const double edge = std::max({hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]});
        const double scale = std::log(0.5 * edge * std::pow(static_cast<double>(count), -1.0 / 3.0));
        const double logit = std::log(0.1 / 0.9);
        for (int i = 0; i < count; ++i) {
            out->means[3 * i] = ux(rng->eng);
            out->means[3 * i + 1] = uy(rng->eng);
            out->means[3 * i + 2] = uz(rng->eng);
            for (int c = 0; c < 3; ++c) {
                out->log_scales[3 * i + c] = scale;
                out->colors[3 * i + c] = ucolor(rng->eng);
            }
            out->rotations[4 * i] = 1.0;
            out->rotations[4 * i + 1] = out->rotations[4 * i + 2] = out->rotations[4 * i + 3] = 0.0;
            out->opacity_logits[i] = logit;
        }
    });
}

int slm_toy_gaussians(int count, uint64_t seed, slm_gaussians* out) {
    return guarded([&] {  // io::generate_toy_scene's ground truth (scene_gen.cpp:38-71)
        if (count < 1) throw std::invalid_argument("toy scene needs at least one Gaussian");
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> upos(-0.8, 0.8);
        std::uniform_real_distribution<double> uscale(std::log(0.12), std::log(0.35));
        std::uniform_real_distribution<double> uquat(-1.0, 1.0);
        std::uniform_real_distribution<double> uopacity(0.4, 0.9);
        std::uniform_real_distribution<double> ucolor(-1.2, 1.2);
        for (int i = 0; i < count; ++i) {
            for (int c = 0; c < 3; ++c) {
                out->means[3 * i + c] = upos(rng);
                out->log_scales[3 * i + c] = uscale(rng);
                out->colors[3 * i + c] = ucolor(rng);
            }
            double q[4], norm = 0.0;
            do {
                norm = 0.0;
                for (double& v : q) {
                    v = uquat(rng);
                    norm += v * v;
                }
            } while (norm < 1e-4);
            const double o = uopacity(rng);
            out->opacity_logits[i] = std::log(o / (1.0 - o));
            // GaussianSet::renormalize_rotations (types.cpp:62-73)
            const double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
            for (int c = 0; c < 4; ++c) out->rotations[4 * i + c] = q[c] / n;
        }
    });
}

int slm_ring_camera(double angle, double radius, double height, int width, int height_px, slm_camera* out) {
    return guarded([&] {  // io::ring_camera (scene_gen.cpp:11-36), W x H allowed
        const double pos[3] = {radius * std::cos(angle), height, radius * std::sin(angle)};
        double fwd[3] = {0.0 - pos[0], 0.0 - pos[1], 0.0 - pos[2]};
        const double fn = std::sqrt(fwd[0] * fwd[0] + fwd[1] * fwd[1] + fwd[2] * fwd[2]);
        for (double& v : fwd) v /= fn;
        double right[3] = {fwd[1] * 0.0 - fwd[2] * 1.0, fwd[2] * 0.0 - fwd[0] * 0.0, fwd[0] * 1.0 - fwd[1] * 0.0};
        const double rn = std::sqrt(right[0] * right[0] + right[1] * right[1] + right[2] * right[2]);
        for (double& v : right) v /= rn;
        const double down[3] = {fwd[1] * right[2] - fwd[2] * right[1], fwd[2] * right[0] - fwd[0] * right[2],
                                fwd[0] * right[1] - fwd[1] * right[0]};
        std::memset(out, 0, sizeof *out);
        for (int k = 0; k < 3; ++k) {
            out->world_to_cam[k] = right[k];
            out->world_to_cam[3 + k] = down[k];
            out->world_to_cam[6 + k] = fwd[k];
        }
        for (int r = 0; r < 3; ++r) {
            const double* row = out->world_to_cam + 3 * r;
            out->translation[r] = -(row[0] * pos[0] + row[1] * pos[1] + row[2] * pos[2]);
        }
        out->width = width;
        out->height = height_px > 0 ? height_px : width;
        const double fov_x = 50.0 * 3.14159265358979323846 / 180.0;
        out->fx = out->fy = 0.5 * width / std::tan(0.5 * fov_x);
        out->cx = 0.5 * width;
        out->cy = 0.5 * out->height;
        out->near_clip = 0.2;
    });
}

}  // extern "C"
