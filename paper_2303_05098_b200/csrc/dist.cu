// Row-partitioned iterated SpMV across ranks (config 5), one
// process (or thread) per GPU, no collective on the data path.  The
// reference's only intra-op parallelism is a row-block partition of one
// multiply over std::threads (spmv.cpp:142-189); here the row partition spans
// GPUs and the x exchange rides on NVLink peer memory:
//
//   SO_DIST_HALO (banded / stencil DIA, window [r0-h, r1+h)): the rows a
//     neighbour needs are computed once and stored twice -- into the local
//     window and straight into the neighbour's window (dia_push_kernel), whose
//     last CTA publishes the iteration number to the neighbour's flag with a
//     release.sys store; the interior rows never wait for anyone.
//   SO_DIST_ALLGATHER (any format, rows [r0, r1) x all columns): the local
//     multiply writes its rows of the next x, then one kernel stores them into
//     every peer's copy of x over peer memory and publishes a flag per peer
//     (an all-gather fused into the epilogue of the iteration).
//
// Every rank owns one peer-shareable block (cudaMalloc, one CUDA IPC handle):
// [x buffer 0 | x buffer 1 | flags], double-buffered by iteration parity.
// WAR safety: a rank writes a peer's buffer for iteration it+1 only after
// that peer published iteration it-1 ... i.e. finished reading that buffer
// (HALO: only the halo rows, read by the boundary kernel that publishes;
// ALLGATHER: the whole buffer, read by the multiply that precedes the
// broadcast).  The P-rank iterate is bitwise equal to the 1-rank iterate:
// no row's summation order changes.
#include <cstring>
#include <string>
#include <vector>

#include "matrix.cuh"

namespace sob {

namespace {

constexpr unsigned long long kDistWaitNs = 60ull * 1000 * 1000 * 1000;
__device__ unsigned long long g_dist_timeouts = 0;

// Wait (acquire, system scope) until every listed flag reaches `value`;
// thread k watches flag k.  Gives up after kDistWaitNs (a dead peer must not
// wedge this GPU) and counts the timeout.
__global__ void wait_flags_kernel(const unsigned long long* flags, int nflags, int skip,
                                  unsigned long long value) {
    const int k = threadIdx.x;
    if (k >= nflags || k == skip) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + k) : "memory");
        if (v >= value) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > kDistWaitNs) {
            atomicAdd(&g_dist_timeouts, 1ull);
            break;
        }
        __nanosleep(200);
    }
}

// rows [0, len) of src -> every peer p's dst[p] (16-byte stores when both
// sides are 16-byte aligned), then the last CTA publishes `value` to each
// peer's flag slot (release, system scope).
__global__ void __launch_bounds__(256)
    bcast_rows_kernel(const double* __restrict__ src, int64_t len, double* const* __restrict__ dst, int npeers,
                      unsigned* ticket, unsigned long long* const* __restrict__ flag, unsigned long long value) {
    __shared__ bool last;
    const int64_t npair = len >> 1;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int p = 0; p < npeers; ++p) {
        double* d = dst[p];
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
        if (vec) {
            for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < npair; j += stride)
                reinterpret_cast<double2*>(d)[j] = reinterpret_cast<const double2*>(src)[j];
            if ((len & 1) && blockIdx.x == 0 && threadIdx.x == 0) d[len - 1] = src[len - 1];
        } else {
            for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < len; j += stride) d[j] = src[j];
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *ticket = 0;
        __threadfence_system();
        for (int p = 0; p < npeers; ++p)
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag[p]), "l"(value) : "memory");
    }
}

}  // namespace

}  // namespace sob

struct so_dist {
    int device = 0;
    int32_t kind = SO_DIST_HALO;
    int32_t rank = 0, world = 1;
    const so_matrix* m = nullptr;  // borrowed: the caller keeps it alive
    std::vector<int64_t> starts;   // [world+1]
    int64_t halo = 0;
    int64_t r0 = 0, r1 = 0, w0 = 0, w1 = 0;  // owned rows, x window (ALLGATHER: [0, n))
    int64_t len = 0;                          // doubles per x buffer
    int nflags = 2;
    void* block = nullptr;                     // [buf0 | buf1 | flags]
    unsigned* tickets = nullptr;               // [2] (own memory, not shared)
    std::vector<void*> opened;                 // peer blocks mapped here
    std::vector<char*> peer;                   // [world] mapped base of each peer's block (null: self/absent)
    double** d_dst = nullptr;                  // ALLGATHER: [2][world-1] peer buffers per parity
    unsigned long long** d_flag = nullptr;     // ALLGATHER: [world-1] peer flag slots for this rank
    bool connected = false;
    int64_t it = 0;

    double* buf(int k) const { return static_cast<double*>(block) + size_t(k) * size_t(len); }
    unsigned long long* flags() const {
        return reinterpret_cast<unsigned long long*>(static_cast<double*>(block) + 2 * size_t(len));
    }
    size_t block_bytes() const { return sizeof(double) * 2 * size_t(len) + sizeof(unsigned long long) * size_t(nflags); }
    int64_t w0_of(int q) const { return kind == SO_DIST_HALO ? std::max<int64_t>(0, starts[q] - halo) : 0; }
    double* peer_buf(int q, int k) const {
        const int64_t qlen = kind == SO_DIST_HALO
                                 ? std::min<int64_t>(starts[world], starts[q + 1] + halo) - w0_of(q)
                                 : len;
        return reinterpret_cast<double*>(peer[size_t(q)]) + size_t(k) * size_t(qlen);
    }
    unsigned long long* peer_flags(int q) const {
        const int64_t qlen = kind == SO_DIST_HALO
                                 ? std::min<int64_t>(starts[world], starts[q + 1] + halo) - w0_of(q)
                                 : len;
        return reinterpret_cast<unsigned long long*>(reinterpret_cast<double*>(peer[size_t(q)]) + 2 * size_t(qlen));
    }
};

using namespace sob;

namespace {

void dist_free_device(so_dist* d) {
    cudaSetDevice(d->device);
    cudaDeviceSynchronize();
    for (void* p : d->opened) cudaIpcCloseMemHandle(p);
    if (d->block) cudaFree(d->block);
    if (d->tickets) cudaFree(d->tickets);
    if (d->d_dst) cudaFree(d->d_dst);
    if (d->d_flag) cudaFree(d->d_flag);
}

}  // namespace

extern "C" {

so_status so_dist_create(const so_matrix* m, int32_t kind, int32_t rank, int32_t world, const int64_t* row_starts,
                         int64_t halo, so_dist** out) {
    return guard([&] {
        if (!m || !row_starts || !out) fail(SO_INVALID_INPUT, "dist_create: null argument");
        *out = nullptr;
        if (kind != SO_DIST_HALO && kind != SO_DIST_ALLGATHER) fail(SO_INVALID_INPUT, "dist_create: unknown kind");
        if (world < 1 || rank < 0 || rank >= world) fail(SO_INVALID_INPUT, "dist_create: rank outside [0, world)");
        if (row_starts[0] != 0) fail(SO_INVALID_INPUT, "dist_create: row_starts[0] must be 0");
        for (int q = 0; q < world; ++q)
            if (row_starts[q + 1] < row_starts[q]) fail(SO_INVALID_INPUT, "dist_create: row_starts must not decrease");
        std::unique_ptr<so_dist> d(new so_dist());
        d->device = m->device;
        d->kind = kind;
        d->rank = rank;
        d->world = world;
        d->m = m;
        d->starts.assign(row_starts, row_starts + world + 1);
        d->halo = halo;
        const int64_t n = row_starts[world];
        d->r0 = row_starts[rank];
        d->r1 = row_starts[rank + 1];
        if (m->nrows != d->r1 - d->r0)
            fail(SO_DIMENSION_MISMATCH, "dist_create: local matrix has " + std::to_string(m->nrows) +
                                            " rows, the partition gives this rank " + std::to_string(d->r1 - d->r0));
        if (kind == SO_DIST_HALO) {
            if (halo < 0) fail(SO_INVALID_INPUT, "dist_create: negative halo");
            if (m->format != SO_DIA && !(m->format == SO_HDC && m->csr.nnz == 0))
                fail(SO_INVALID_INPUT, "dist_create: halo exchange needs a DIA-window matrix (DIA, or HDC with an "
                                       "empty CSR part); use SO_DIST_ALLGATHER");
            for (int q = 0; q < world && world > 1; ++q)
                if (row_starts[q + 1] - row_starts[q] < 2 * halo)
                    fail(SO_INVALID_INPUT, "dist_create: every rank needs >= 2*halo rows (fewer ranks)");
            d->w0 = std::max<int64_t>(0, d->r0 - halo);
            d->w1 = std::min<int64_t>(n, d->r1 + halo);
            d->nflags = 2;  // [0] from the left neighbour, [1] from the right
        } else {
            d->w0 = 0;
            d->w1 = n;
            d->nflags = std::max(2, int(world));  // [q] from rank q
        }
        if (m->ncols != d->w1 - d->w0)
            fail(SO_DIMENSION_MISMATCH, "dist_create: local matrix has " + std::to_string(m->ncols) +
                                            " columns, its x window has " + std::to_string(d->w1 - d->w0));
        d->len = d->w1 - d->w0;
        SOB_CUDA(cudaSetDevice(d->device));
        const cudaError_t e = cudaMalloc(&d->block, d->block_bytes());  // IPC needs a plain cudaMalloc
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            fail(SO_OUT_OF_MEMORY, "dist_create: out of device memory");
        }
        SOB_CUDA(e);
        SOB_CUDA(cudaMemset(d->block, 0, d->block_bytes()));
        SOB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d->tickets), 2 * sizeof(unsigned)));
        SOB_CUDA(cudaMemset(d->tickets, 0, 2 * sizeof(unsigned)));
        d->peer.assign(size_t(world), nullptr);
        *out = d.release();
    });
}

so_status so_dist_handle(const so_dist* d, so_ipc_handle* out) {
    return guard([&] {
        if (!d || !out) fail(SO_INVALID_INPUT, "dist_handle: null argument");
        SOB_CUDA(cudaSetDevice(d->device));
        cudaIpcMemHandle_t h;
        SOB_CUDA(cudaIpcGetMemHandle(&h, d->block));
        static_assert(sizeof(h) <= sizeof(out->bytes), "IPC handle size");
        std::memset(out->bytes, 0, sizeof(out->bytes));
        std::memcpy(out->bytes, &h, sizeof(h));
    });
}

so_status so_dist_connect(so_dist* d, const so_ipc_handle* handles) {
    return guard([&] {
        SOB_RANGE("so_dist_connect");
        if (!d || (!handles && d->world > 1)) fail(SO_INVALID_INPUT, "dist_connect: null argument");
        if (d->connected) fail(SO_INVALID_INPUT, "dist_connect: already connected");
        SOB_CUDA(cudaSetDevice(d->device));
        std::vector<int> need;
        if (d->kind == SO_DIST_HALO) {
            if (d->rank > 0) need.push_back(d->rank - 1);
            if (d->rank < d->world - 1) need.push_back(d->rank + 1);
        } else {
            for (int q = 0; q < d->world; ++q)
                if (q != d->rank) need.push_back(q);
        }
        for (int q : need) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handles[q].bytes, sizeof(h));
            void* p = nullptr;
            SOB_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            d->opened.push_back(p);
            d->peer[size_t(q)] = static_cast<char*>(p);
        }
        if (d->kind == SO_DIST_ALLGATHER && d->world > 1) {
            const int np = d->world - 1;
            std::vector<double*> dst(static_cast<size_t>(2 * np));
            std::vector<unsigned long long*> fl(static_cast<size_t>(np));
            int k = 0;
            for (int q : need) {
                dst[size_t(k)] = d->peer_buf(q, 0) + d->r0;
                dst[size_t(np + k)] = d->peer_buf(q, 1) + d->r0;
                fl[size_t(k)] = d->peer_flags(q) + d->rank;
                ++k;
            }
            SOB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d->d_dst), dst.size() * sizeof(double*)));
            SOB_CUDA(cudaMemcpy(d->d_dst, dst.data(), dst.size() * sizeof(double*), cudaMemcpyHostToDevice));
            SOB_CUDA(cudaMalloc(reinterpret_cast<void**>(&d->d_flag), fl.size() * sizeof(unsigned long long*)));
            SOB_CUDA(cudaMemcpy(d->d_flag, fl.data(), fl.size() * sizeof(unsigned long long*), cudaMemcpyHostToDevice));
        }
        d->connected = true;
    });
}

so_status so_dist_x(const so_dist* d, int32_t which, double** x_dev, int64_t* offset, int64_t* len) {
    return guard([&] {
        if (!d || !x_dev) fail(SO_INVALID_INPUT, "dist_x: null argument");
        const int k = which < 0 ? int(d->it % 2) : (which & 1);
        *x_dev = d->buf(k);
        if (offset) *offset = d->w0;
        if (len) *len = d->len;
    });
}

so_status so_dist_iterate(so_dist* d, int64_t iters, void* stream) {
    return guard([&] {
        SOB_RANGE("so_dist_iterate");
        if (!d) fail(SO_INVALID_INPUT, "dist_iterate: null argument");
        if (!d->connected && d->world > 1) fail(SO_INVALID_INPUT, "dist_iterate: not connected");
        if (iters < 0) fail(SO_INVALID_INPUT, "dist_iterate: negative iteration count");
        SOB_CUDA(cudaSetDevice(d->device));
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx(d->device).stream;
        const so_matrix& m = *d->m;
        const int64_t nloc = d->r1 - d->r0;
        const int64_t own_lo = d->r0 - d->w0;
        const bool left = d->rank > 0, right = d->rank < d->world - 1;
        for (int64_t k = 0; k < iters; ++k) {
            const int64_t it = d->it;
            const int c = int(it % 2), nx = int((it + 1) % 2);
            double* cur = d->buf(c);
            double* y = d->buf(nx) + own_lo;
            if (d->kind == SO_DIST_HALO) {
                // my halo of `cur` was pushed by the neighbours during iteration it-1
                const int64_t lo = left ? std::min(d->halo, nloc) : 0;
                const int64_t hi = right ? std::max(nloc - d->halo, lo) : nloc;
                if (d->world > 1) {
                    wait_flags_kernel<<<1, 32, 0, s>>>(d->flags(), 2, left ? (right ? -1 : 1) : 0,
                                                        (unsigned long long)it);
                    SOB_LAUNCH("wait_flags_kernel");
                }
                if (left && lo > 0) {  // first h rows -> left neighbour's right halo
                    const int q = d->rank - 1;
                    double* remote = d->peer_buf(q, nx) + (d->r0 - d->w0_of(q));
                    spmv_rows_push(m, cur, y, 0, lo, remote, d->tickets, d->peer_flags(q) + 1,
                                   (unsigned long long)(it + 1), s);
                }
                if (right && hi < nloc) {  // last h rows -> right neighbour's left halo
                    const int q = d->rank + 1;
                    double* remote = d->peer_buf(q, nx) + (d->r0 + hi - d->w0_of(q));
                    spmv_rows_push(m, cur, y, hi, nloc, remote, d->tickets + 1, d->peer_flags(q) + 0,
                                   (unsigned long long)(it + 1), s);
                }
                if (hi > lo) spmv_device_rows(m, cur, y, lo, hi, s);
            } else {
                if (d->world > 1) {
                    wait_flags_kernel<<<1, 64, 0, s>>>(d->flags(), d->world, d->rank, (unsigned long long)it);
                    SOB_LAUNCH("wait_flags_kernel");
                }
                if (nloc > 0) spmv_device(m, cur, y, s);
                if (d->world > 1) {
                    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(nloc, 512), 4 * 148)));
                    bcast_rows_kernel<<<grid, 256, 0, s>>>(y, nloc, d->d_dst + size_t(nx) * size_t(d->world - 1),
                                                           d->world - 1, d->tickets, d->d_flag,
                                                           (unsigned long long)(it + 1));
                    SOB_LAUNCH("bcast_rows_kernel");
                }
            }
            d->it = it + 1;
        }
    });
}

int64_t so_dist_timeouts(void) {
    unsigned long long v = 0;
    const so_status st = guard([&] { SOB_CUDA(cudaMemcpyFromSymbol(&v, g_dist_timeouts, sizeof(v))); });
    return st == SO_OK ? int64_t(v) : -1;
}

void so_dist_free(so_dist* d) {
    if (!d) return;
    dist_free_device(d);
    delete d;
}

}  // extern "C"
