// Context lifecycle and the host-buffer end-to-end entry of include/gnna.h.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "gnna_common.cuh"

namespace gnna {

// ------------------------------------------------ pageable host transfers
// cudaMemcpy from pageable memory is staged by the driver through its own
// pinned buffer on one thread (~11 GB/s here).  Large pageable copies go
// through the context's ring of pinned chunks instead: host threads copy
// chunk k + 1 into its bounce buffer while the DMA engine moves chunk k.
// Pinned (registered) host memory is copied directly, as before.
struct HostPool {
    explicit HostPool(unsigned n) : n_(n) {
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    unsigned size() const { return n_; }
    // f(worker) on every worker; returns when all are done
    void run(const std::function<void(unsigned)>& f) {
        {
            std::lock_guard<std::mutex> l(m_);
            job_ = &f;
            pending_ = n_;
            ++gen_;
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [&] { return pending_ == 0; });
    }

private:
    void loop(unsigned i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* f;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = job_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> l(m_);
            if (--pending_ == 0) done_.notify_all();
        }
    }
    unsigned n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* job_ = nullptr;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
};

struct Staging {
    static constexpr size_t CH = 8u << 20;  // bytes per bounce buffer
    static constexpr int SLOTS = 3;
    void* buf[SLOTS] = {};
    cudaEvent_t ev[SLOTS] = {};
    bool busy[SLOTS] = {};
    HostPool pool;
    explicit Staging(unsigned threads) : pool(threads) {
        for (int i = 0; i < SLOTS; ++i) {
            GNNA_CUDA(cudaHostAlloc(&buf[i], CH, cudaHostAllocDefault));
            GNNA_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~Staging() {
        for (int i = 0; i < SLOTS; ++i) {
            if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
    // memcpy split over the pool's threads in 64-byte aligned parts
    void pmemcpy(void* dst, const void* src, size_t len) {
        const unsigned n = pool.size();
        const size_t part = ((len + n - 1) / n + 63) & ~size_t(63);
        pool.run([&](unsigned i) {
            const size_t b = (size_t)i * part;
            if (b < len)
                std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, std::min(part, len - b));
        });
    }
};

constexpr size_t kStageMin = 4u << 20;  // smaller copies: the driver's own staging

bool pageable(const void* p) {
    static const bool off = [] {
        const char* e = std::getenv("GNNA_STAGING");  // A/B switch (0: the driver's staging)
        return e && *e == '0';
    }();
    if (off) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

Staging& staging(gnna_ctx* ctx) {
    if (!ctx->staging) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        ctx->staging = new Staging(std::min(8u, hw));
    }
    return *ctx->staging;
}

// Host -> device, stream-ordered on ctx->stream; the host source may be
// reused as soon as this returns.
void copy_h2d(gnna_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
    if (!bytes) return;
    if (bytes < kStageMin || !pageable(h_src)) {
        // (a pageable source is free again on return: the driver stages it before returning)
        GNNA_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        return;
    }
    Staging& st = staging(ctx);
    for (size_t off = 0, k = 0; off < bytes; off += Staging::CH, ++k) {
        const int s = (int)(k % Staging::SLOTS);
        const size_t len = std::min(Staging::CH, bytes - off);
        if (st.busy[s]) GNNA_CUDA(cudaEventSynchronize(st.ev[s]));
        st.pmemcpy(st.buf[s], static_cast<const char*>(h_src) + off, len);
        GNNA_CUDA(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, st.buf[s], len, cudaMemcpyHostToDevice, ctx->stream));
        GNNA_CUDA(cudaEventRecord(st.ev[s], ctx->stream));
        st.busy[s] = true;
    }
}

// Device -> host after the work already queued on ctx->stream; returns when
// the host buffer holds the data.
void copy_d2h(gnna_ctx* ctx, void* h_dst, const void* d_src, size_t bytes) {
    if (bytes < kStageMin || !pageable(h_dst)) {
        if (bytes) GNNA_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        GNNA_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    Staging& st = staging(ctx);
    const size_t chunks = (bytes + Staging::CH - 1) / Staging::CH;
    auto dma = [&](size_t k) {
        const int s = (int)(k % Staging::SLOTS);
        const size_t off = k * Staging::CH, len = std::min(Staging::CH, bytes - off);
        if (st.busy[s]) GNNA_CUDA(cudaEventSynchronize(st.ev[s]));
        GNNA_CUDA(cudaMemcpyAsync(st.buf[s], static_cast<const char*>(d_src) + off, len, cudaMemcpyDeviceToHost,
                                  ctx->stream));
        GNNA_CUDA(cudaEventRecord(st.ev[s], ctx->stream));
        st.busy[s] = true;
    };
    for (size_t k = 0; k < chunks && k < (size_t)Staging::SLOTS; ++k) dma(k);
    for (size_t k = 0; k < chunks; ++k) {
        const int s = (int)(k % Staging::SLOTS);
        const size_t off = k * Staging::CH, len = std::min(Staging::CH, bytes - off);
        GNNA_CUDA(cudaEventSynchronize(st.ev[s]));
        st.pmemcpy(static_cast<char*>(h_dst) + off, st.buf[s], len);
        st.busy[s] = false;
        if (k + Staging::SLOTS < chunks) dma(k + Staging::SLOTS);
    }
}

void validate_params(const gnna_params* p);
void aggregate_plan(gnna_ctx* ctx, const gnna_plan* plan, int dtype, int dim_mode, const void* x, void* y,
                    uint32_t epi, const float* scale, double alpha);
void cost_report(gnna_ctx* ctx, const gnna_plan* plan, int dim_mode, uint64_t line, uint64_t cache_cap,
                 uint64_t cache_line, gnna_cost* out);
void rebase_u64(gnna_ctx* ctx, uint64_t* v, uint64_t count, uint64_t base);
}  // namespace gnna

extern "C" {

const char* gnna_version(void) { return "gnna-b200 0.1 (sm_100a)"; }

gnna_status gnna_create(int device, gnna_ctx** out) {
    return gnna::guard(nullptr, [&] {
        if (!out) gnna::raise(GNNA_ERR_DOMAIN, "null output pointer");
        int count = 0;
        GNNA_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) gnna::raise(GNNA_ERR_CUDA, "no such CUDA device");
        int major = 0, minor = 0;
        GNNA_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        GNNA_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
        if (major != 10 || minor != 0)
            gnna::raise(GNNA_ERR_CUDA, "libgnna is built for sm_100a (B200); device is sm_" +
                                           std::to_string(major) + std::to_string(minor));
        GNNA_CUDA(cudaSetDevice(device));
        // Scratch buffers come from the stream-ordered pool.  Its default
        // release threshold (0) hands memory back to the OS at every stream
        // sync, so the next cudaMallocAsync re-maps it (~100 us per call on
        // large buffers); keep freed memory cached in the pool instead.
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        auto ctx = new gnna_ctx();
        ctx->device = device;
        cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
        cudaDeviceGetAttribute(&ctx->l2_bytes, cudaDevAttrL2CacheSize, device);
        cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        *out = ctx;
    });
}

void gnna_destroy(gnna_ctx* ctx) { delete ctx; }

}  // extern "C"

gnna_ctx::~gnna_ctx() {
    if (staging) {
        cudaStreamSynchronize(stream);
        delete staging;
    }
}

extern "C" {

gnna_status gnna_set_stream(gnna_ctx* ctx, void* stream) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        ctx->stream = static_cast<cudaStream_t>(stream);
    });
}

void* gnna_get_stream(const gnna_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

gnna_status gnna_synchronize(gnna_ctx* ctx) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        GNNA_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

const char* gnna_last_error(const gnna_ctx* ctx) { return ctx ? ctx->err.c_str() : "null gnna_ctx"; }

gnna_status gnna_set_l2_window(gnna_ctx* ctx, const void* base, uint64_t bytes, double hit_ratio,
                               uint64_t* applied) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (hit_ratio < 0.0 || hit_ratio > 1.0) gnna::raise(GNNA_ERR_DOMAIN, "set_l2_window: hit_ratio in [0, 1]");
        // the persisting-L2 limit is a property of the current device: make it the context's
        int prev = 0;
        GNNA_CUDA(cudaGetDevice(&prev));
        struct Restore {
            int d;
            ~Restore() { cudaSetDevice(d); }
        } restore{prev};
        GNNA_CUDA(cudaSetDevice(ctx->device));
        cudaStreamAttrValue v{};
        if (!bytes || !base) {
            v.accessPolicyWindow.num_bytes = 0;
            GNNA_CUDA(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v));
            GNNA_CUDA(cudaCtxResetPersistingL2Cache());
            GNNA_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
            if (applied) *applied = 0;
            return;
        }
        int max_persist = 0, max_window = 0;
        GNNA_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
        GNNA_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device));
        const uint64_t win = std::min<uint64_t>(bytes, (uint64_t)std::max(0, max_window));
        const uint64_t carve = std::min<uint64_t>(win, (uint64_t)std::max(0, max_persist));
        GNNA_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
        v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
        v.accessPolicyWindow.num_bytes = win;
        v.accessPolicyWindow.hitRatio = (float)hit_ratio;
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        GNNA_CUDA(cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v));
        if (applied) *applied = win;
    });
}

uint64_t gnna_launch_count(const gnna_ctx* ctx) { return ctx ? ctx->launches : 0; }

gnna_status gnna_device_alloc(gnna_ctx* ctx, size_t bytes, void** out) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (!out) gnna::raise(GNNA_ERR_DOMAIN, "null output pointer");
        *out = nullptr;
        GNNA_CUDA(cudaMallocAsync(out, bytes ? bytes : 1, ctx->stream));
    });
}

gnna_status gnna_device_free(gnna_ctx* ctx, void* p) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        if (p) GNNA_CUDA(cudaFreeAsync(p, ctx->stream));
    });
}

gnna_status gnna_copy_to_device(gnna_ctx* ctx, void* d_dst, const void* h_src, size_t bytes) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::copy_h2d(ctx, d_dst, h_src, bytes);
    });
}

gnna_status gnna_copy_to_host(gnna_ctx* ctx, void* h_dst, const void* d_src, size_t bytes) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::copy_d2h(ctx, h_dst, d_src, bytes);
    });
}

gnna_status gnna_aggregate_host_rows(gnna_ctx* ctx, int dtype, const uint64_t* h_row_ptr, const uint32_t* h_col,
                                     uint32_t n, uint32_t row_begin, uint32_t row_end, const gnna_params* p,
                                     int strategy, int dim_mode, const void* h_x, void* h_y, uint64_t line_bytes,
                                     uint64_t cache_capacity, uint64_t cache_line, gnna_cost* cost) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::validate_params(p);
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        if (row_begin > row_end || row_end > n) gnna::raise(GNNA_ERR_DOMAIN, "aggregate_host: bad row range");
        cudaStream_t s = ctx->stream;
        const uint32_t rows = row_end - row_begin;
        const uint64_t e0 = h_row_ptr[row_begin], e1 = h_row_ptr[row_end];
        const uint64_t nnz = e1 - e0;
        const size_t elem = dtype == GNNA_F32 ? 4 : 8;
        const size_t xbytes = (size_t)n * p->dim * elem;
        const size_t ybytes = (size_t)rows * p->dim * elem;
        // The shard is a rows x n CSR: its own rebased row_ptr and column
        // slice, gathering from the full (replicated) feature matrix.
        gnna::DevBuf<uint64_t> rp((uint64_t)rows + 1, s);
        gnna::DevBuf<uint32_t> col(nnz ? nnz : 1, s);
        gnna::DevBuf<uint8_t> x(xbytes ? xbytes : 1, s), y(ybytes ? ybytes : 1, s);
        GNNA_CUDA(cudaMemcpyAsync(rp.get(), h_row_ptr + row_begin, ((size_t)rows + 1) * 8, cudaMemcpyHostToDevice, s));
        if (e0) gnna::rebase_u64(ctx, rp.get(), (uint64_t)rows + 1, e0);
        gnna::copy_h2d(ctx, col.get(), h_col + e0, nnz * 4);
        gnna::copy_h2d(ctx, x.get(), h_x, xbytes);
        gnna_plan* plan = nullptr;
        gnna_status st = gnna_plan_create(ctx, rp.get(), col.get(), rows, 0, rows, p, strategy, &plan);
        if (st != GNNA_OK) gnna::raise(st, ctx->err);
        try {
            gnna::aggregate_plan(ctx, plan, dtype, dim_mode, x.get(), y.get(), 0, nullptr, 0.0);
            if (cost) gnna::cost_report(ctx, plan, dim_mode, line_bytes, cache_capacity, cache_line, cost);
            gnna::copy_d2h(ctx, h_y, y.get(), ybytes);
        } catch (...) {
            gnna_plan_destroy(plan);
            throw;
        }
        gnna_plan_destroy(plan);
    });
}

gnna_status gnna_aggregate_host_stream(gnna_ctx* ctx, int dtype, const gnna_params* p, int strategy, int dim_mode,
                                       const gnna_host_batch* batches, uint32_t num_batches) {
    return gnna::guard(ctx, [&] {
        gnna::require_ctx(ctx);
        gnna::validate_params(p);
        if (dtype != GNNA_F32 && dtype != GNNA_F64) gnna::raise(GNNA_ERR_DOMAIN, "unknown dtype");
        if (!num_batches) return;
        if (!batches) gnna::raise(GNNA_ERR_DOMAIN, "null batches");
        const size_t elem = dtype == GNNA_F32 ? 4 : 8;
        // capacity of one device buffer set = max over the batches
        uint64_t max_rows = 0, max_nnz = 0, max_x = 0;
        for (uint32_t i = 0; i < num_batches; ++i) {
            const gnna_host_batch& b = batches[i];
            if (b.row_begin > b.row_end || b.row_end > b.n) gnna::raise(GNNA_ERR_DOMAIN, "aggregate_host: bad row range");
            max_rows = std::max<uint64_t>(max_rows, b.row_end - b.row_begin);
            max_nnz = std::max<uint64_t>(max_nnz, b.h_row_ptr[b.row_end] - b.h_row_ptr[b.row_begin]);
            max_x = std::max<uint64_t>(max_x, (uint64_t)b.n * p->dim * elem);
        }
        cudaStream_t cs = ctx->stream, up = nullptr, down = nullptr;
        GNNA_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
        GNNA_CUDA(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
        struct Slot {
            gnna::DevBuf<uint64_t> rp;
            gnna::DevBuf<uint32_t> col;
            gnna::DevBuf<uint8_t> x, y;
            cudaEvent_t uploaded = nullptr, computed = nullptr, downloaded = nullptr;
        } slot[2];
        auto cleanup = [&] {
            cudaStreamSynchronize(up);
            cudaStreamSynchronize(down);
            cudaStreamSynchronize(cs);
            for (auto& s : slot) {
                if (s.uploaded) cudaEventDestroy(s.uploaded);
                if (s.computed) cudaEventDestroy(s.computed);
                if (s.downloaded) cudaEventDestroy(s.downloaded);
            }
            cudaStreamDestroy(up);
            cudaStreamDestroy(down);
        };
        try {
            for (auto& s : slot) {
                s.rp = gnna::DevBuf<uint64_t>(max_rows + 1, cs);
                s.col = gnna::DevBuf<uint32_t>(max_nnz ? max_nnz : 1, cs);
                s.x = gnna::DevBuf<uint8_t>(max_x ? max_x : 1, cs);
                s.y = gnna::DevBuf<uint8_t>(max_rows * p->dim * elem + 1, cs);
                GNNA_CUDA(cudaEventCreateWithFlags(&s.uploaded, cudaEventDisableTiming));
                GNNA_CUDA(cudaEventCreateWithFlags(&s.computed, cudaEventDisableTiming));
                GNNA_CUDA(cudaEventCreateWithFlags(&s.downloaded, cudaEventDisableTiming));
                // start "free": nothing to wait for
                GNNA_CUDA(cudaEventRecord(s.computed, cs));
                GNNA_CUDA(cudaEventRecord(s.downloaded, cs));
            }
            GNNA_CUDA(cudaStreamSynchronize(cs));  // buffers allocated before the copy streams use them
            auto upload = [&](uint32_t i) {
                const gnna_host_batch& b = batches[i];
                Slot& s = slot[i & 1];
                const uint32_t rows = b.row_end - b.row_begin;
                const uint64_t e0 = b.h_row_ptr[b.row_begin], nnz = b.h_row_ptr[b.row_end] - e0;
                GNNA_CUDA(cudaStreamWaitEvent(up, s.computed, 0));  // slot's previous batch done reading
                GNNA_CUDA(cudaMemcpyAsync(s.rp.get(), b.h_row_ptr + b.row_begin, ((size_t)rows + 1) * 8,
                                          cudaMemcpyHostToDevice, up));
                if (nnz) GNNA_CUDA(cudaMemcpyAsync(s.col.get(), b.h_col + e0, nnz * 4, cudaMemcpyHostToDevice, up));
                const size_t xb = (size_t)b.n * p->dim * elem;
                if (xb) GNNA_CUDA(cudaMemcpyAsync(s.x.get(), b.h_x, xb, cudaMemcpyHostToDevice, up));
                GNNA_CUDA(cudaEventRecord(s.uploaded, up));
            };
            upload(0);
            for (uint32_t i = 0; i < num_batches; ++i) {
                const gnna_host_batch& b = batches[i];
                Slot& s = slot[i & 1];
                if (i + 1 < num_batches) upload(i + 1);  // keep the H2D engine busy
                const uint32_t rows = b.row_end - b.row_begin;
                const uint64_t e0 = b.h_row_ptr[b.row_begin];
                GNNA_CUDA(cudaStreamWaitEvent(cs, s.uploaded, 0));
                GNNA_CUDA(cudaStreamWaitEvent(cs, s.downloaded, 0));  // y slot free
                if (e0) gnna::rebase_u64(ctx, s.rp.get(), (uint64_t)rows + 1, e0);
                gnna_plan* plan = nullptr;
                gnna_status st = gnna_plan_create(ctx, s.rp.get(), s.col.get(), rows, 0, rows, p, strategy, &plan);
                if (st != GNNA_OK) gnna::raise(st, ctx->err);
                try {
                    gnna::aggregate_plan(ctx, plan, dtype, dim_mode, s.x.get(), s.y.get(), 0, nullptr, 0.0);
                } catch (...) {
                    gnna_plan_destroy(plan);
                    throw;
                }
                GNNA_CUDA(cudaEventRecord(s.computed, cs));
                gnna_plan_destroy(plan);  // stream-ordered frees
                GNNA_CUDA(cudaStreamWaitEvent(down, s.computed, 0));
                const size_t yb = (size_t)rows * p->dim * elem;
                if (yb) GNNA_CUDA(cudaMemcpyAsync(b.h_y, s.y.get(), yb, cudaMemcpyDeviceToHost, down));
                GNNA_CUDA(cudaEventRecord(s.downloaded, down));
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

gnna_status gnna_aggregate_host(gnna_ctx* ctx, int dtype, const uint64_t* h_row_ptr, const uint32_t* h_col,
                                uint32_t n, const gnna_params* p, int strategy, int dim_mode, const void* h_x,
                                void* h_y, uint64_t line_bytes, uint64_t cache_capacity, uint64_t cache_line,
                                gnna_cost* cost) {
    return gnna_aggregate_host_rows(ctx, dtype, h_row_ptr, h_col, n, 0, n, p, strategy, dim_mode, h_x, h_y,
                                    line_bytes, cache_capacity, cache_line, cost);
}

}  // extern "C"
