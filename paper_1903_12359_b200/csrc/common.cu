// common.cu -- errors, device-wide scans, stable counting sort.
#include <mutex>
#include <atomic>

#include "common.cuh"

#include <cstring>
#include <vector>

namespace pgcp {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

const char* get_error() { return g_err.c_str(); }

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(); }

// ---------------------------------------------------------------------------
// scans

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class T>
__global__ void k_tile_sums(const T* __restrict__ in, int64_t n, int64_t* __restrict__ sums) {
    __shared__ int64_t wsum[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        int64_t i = base + j;
        if (i < n) acc += (int64_t)in[i];
    }
    acc = warp_sum_ll(acc);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < SCAN_THREADS / 32; ++w) t += wsum[w];
        sums[blockIdx.x] = t;
    }
}

template <class T>
__global__ void k_tile_scan(const T* __restrict__ in, int64_t n, const int64_t* __restrict__ tile_off,
                            int64_t* __restrict__ out) {
    __shared__ int64_t wsum[SCAN_THREADS / 32];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS];
    int64_t acc = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        int64_t i = base + j;
        v[j] = (i < n) ? (int64_t)in[i] : 0;
        acc += v[j];
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int64_t wpre = 0;
    for (int k = 0; k < w; ++k) wpre += wsum[k];
    int64_t run = tile_off[blockIdx.x] + wpre + inc - acc;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        int64_t i = base + j;
        if (i < n) out[i] = run;
        run += v[j];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == SCAN_THREADS - 1) {
        out[n] = run;  // total
    }
}

template <class T>
int scan_impl(const T* in, int64_t* out, int64_t n, cudaStream_t s) {
    if (n <= 0) {
        PGCP_TRY_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
        return PGCP_OK;
    }
    int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    DevBuf<int64_t> sums, offs;
    PGCP_TRY(sums.alloc(tiles, s));
    PGCP_TRY(offs.alloc(tiles + 1, s));
    k_tile_sums<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, sums.p);
    PGCP_LAUNCH_CHECK();
    if (tiles == 1) {
        PGCP_TRY_CUDA(cudaMemsetAsync(offs.p, 0, sizeof(int64_t), s));
    } else {
        PGCP_TRY(scan_impl<int64_t>(sums.p, offs.p, tiles, s));
    }
    k_tile_scan<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, offs.p, out);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

}  // namespace

int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    return scan_impl<int64_t>(in, out, n, s);
}
int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    return scan_impl<int32_t>(in, out, n, s);
}

// ---------------------------------------------------------------------------
// stable counting sort (one warp owns one tile; no atomics in the scatter)

namespace {

__global__ void k_csort_count(const int32_t* __restrict__ keys, int64_t n, int64_t tile, int64_t ntiles,
                              int32_t* __restrict__ cnt) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < ntiles; t += nwarps) {
        int64_t lo = t * tile, hi = min(lo + tile, n);
        for (int64_t c = lo; c < hi; c += 32) {
            int64_t i = c + lane;
            int key = (i < hi) ? keys[i] : -1;
            unsigned mask = __match_any_sync(0xffffffffu, key);
            int leader = __ffs(mask) - 1;
            if (key >= 0 && lane == leader) cnt[(int64_t)key * ntiles + t] += __popc(mask);
            __syncwarp();
        }
    }
}

__global__ void k_csort_scatter(const int32_t* __restrict__ keys, int64_t n, int64_t tile, int64_t ntiles,
                                int64_t* __restrict__ cursor, int32_t* __restrict__ perm) {
    int lane = threadIdx.x & 31;
    unsigned lt = (1u << lane) - 1u;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < ntiles; t += nwarps) {
        int64_t lo = t * tile, hi = min(lo + tile, n);
        for (int64_t c = lo; c < hi; c += 32) {
            int64_t i = c + lane;
            int key = (i < hi) ? keys[i] : -1;
            unsigned mask = __match_any_sync(0xffffffffu, key);
            int leader = __ffs(mask) - 1;
            int64_t slot = (key >= 0) ? (int64_t)key * ntiles + t : 0;
            int64_t old = (key >= 0 && lane == leader) ? cursor[slot] : 0;
            old = __shfl_sync(0xffffffffu, old, leader);
            if (key >= 0) {
                perm[old + __popc(mask & lt)] = (int32_t)i;
                if (lane == leader) cursor[slot] = old + __popc(mask);
            }
            __syncwarp();
        }
    }
}

__global__ void k_csort_keyoff(const int64_t* __restrict__ cursor0, int32_t nkeys, int64_t ntiles, int64_t n,
                               int64_t* __restrict__ key_off) {
    GRID_STRIDE(k, (int64_t)nkeys + 1) {
        key_off[k] = (k == nkeys) ? n : cursor0[k * ntiles];
    }
}

}  // namespace

int stable_counting_sort(const int32_t* keys, int64_t n, int32_t nkeys, int32_t* perm, int64_t* key_off,
                         cudaStream_t s) {
    if (nkeys <= 0) {
        set_error("stable_counting_sort: nkeys must be positive");
        return PGCP_E_INVALID;
    }
    int64_t tile = 1024;
    while ((int64_t)nkeys * ((n + tile - 1) / tile) > (int64_t)64 << 20) tile *= 2;
    int64_t ntiles = (n + tile - 1) / tile;
    if (ntiles < 1) ntiles = 1;
    int64_t ncnt = (int64_t)nkeys * ntiles;
    DevBuf<int32_t> cnt;
    DevBuf<int64_t> cur;
    PGCP_TRY(cnt.alloc(ncnt, s));
    PGCP_TRY(cnt.zero(s));
    PGCP_TRY(cur.alloc(ncnt + 1, s));
    int block = 256;
    int64_t warps_needed = ntiles;
    int grid = (int)std::min<int64_t>((warps_needed * 32 + block - 1) / block, 148 * 32);
    if (grid < 1) grid = 1;
    if (n > 0) {
        k_csort_count<<<grid, block, 0, s>>>(keys, n, tile, ntiles, cnt.p);
        PGCP_LAUNCH_CHECK();
    }
    PGCP_TRY(exclusive_scan_i32_to_i64(cnt.p, cur.p, ncnt, s));
    k_csort_keyoff<<<grid_for(nkeys + 1, 256), 256, 0, s>>>(cur.p, nkeys, ntiles, n, key_off);
    PGCP_LAUNCH_CHECK();
    if (n > 0) {
        k_csort_scatter<<<grid, block, 0, s>>>(keys, n, tile, ntiles, cur.p, perm);
        PGCP_LAUNCH_CHECK();
    }
    return PGCP_OK;
}

namespace {
// Pinned staging buffers are process-wide and never freed: a host thread
// takes one on its first read and hands it back to the free list when it
// exits. (cudaMallocHost / cudaFreeHost per thread cost a page-pinning call
// and a device-wide synchronisation every time the pipeline's short-lived
// worker threads came and went: 0.1-0.5 s outliers in the flatten and the
// Dirichlet preparation.)
struct PinBuf {
    unsigned char* buf = nullptr;
    size_t cap = 0;
};
std::mutex g_pin_mu;
std::vector<PinBuf> g_pin_free;

struct PinStage {
    unsigned char* buf = nullptr;
    size_t cap = 0, used = 0;
    struct Pending {
        void* host;
        size_t off, bytes;
    };
    std::vector<Pending> pend;
    ~PinStage() {
        if (!buf) return;
        std::lock_guard<std::mutex> lock(g_pin_mu);
        g_pin_free.push_back({buf, cap});
    }
    // a buffer of at least `bytes`: the largest free one if it fits, else a new one
    int take(size_t bytes) {
        {
            std::lock_guard<std::mutex> lock(g_pin_mu);
            if (buf) g_pin_free.push_back({buf, cap});  // too small: back to the list
            buf = nullptr;
            cap = 0;
            int best = -1;
            for (int i = 0; i < (int)g_pin_free.size(); ++i)
                if (g_pin_free[i].cap >= bytes && (best < 0 || g_pin_free[i].cap < g_pin_free[best].cap)) best = i;
            if (best >= 0) {
                buf = g_pin_free[best].buf;
                cap = g_pin_free[best].cap;
                g_pin_free.erase(g_pin_free.begin() + best);
                return PGCP_OK;
            }
        }
        const size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
        PGCP_TRY_CUDA(cudaMallocHost((void**)&buf, want));
        cap = want;
        return PGCP_OK;
    }
};
thread_local PinStage g_pin;
}  // namespace

int d2h_async(void* host, const void* dev, size_t bytes, cudaStream_t s) {
    PinStage& p = g_pin;
    const size_t off = (p.used + 15) & ~(size_t)15;
    if (off + bytes > p.cap) {
        if (!p.pend.empty()) PGCP_TRY(d2h_flush(s));  // queued copies go out first
        if (bytes > p.cap) PGCP_TRY(p.take(bytes));
        return d2h_async(host, dev, bytes, s);
    }
    PGCP_TRY_CUDA(cudaMemcpyAsync(p.buf + off, dev, bytes, cudaMemcpyDeviceToHost, s));
    p.pend.push_back({host, off, bytes});
    p.used = off + bytes;
    return PGCP_OK;
}

int d2h_flush(cudaStream_t s) {
    PinStage& p = g_pin;
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    for (const auto& q : p.pend) memcpy(q.host, p.buf + q.off, q.bytes);
    p.pend.clear();
    p.used = 0;
    return PGCP_OK;
}

}  // namespace pgcp
