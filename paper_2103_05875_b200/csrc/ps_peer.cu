// Peer-memory exchanges of the slab-sharded frame, replacing
// the NCCL all-reduce of the change bitmaps and the send/recv gather of the
// selected cores:
//
//   * ps_detect_changed_bcast (ps_detect.cu): the detect kernel ORs each
//     bitmap word it finds straight into every rank's bitmap (system-scope
//     atomics over NVLink) -- detection and the all-gather in one kernel;
//   * ps_export_tiles_peer: each rank copies its own selected probes' cores
//     into the encoder rank's update atlas at their slots (plain stores to
//     the encoder's memory), commits its blocks and stamps every entry --
//     build and gather in one kernel, no staging payload, no import pass;
//   * ps_peer_signal / ps_peer_wait: release / acquire flags (system scope)
//     that order those stores with the consumers on the other GPUs;
//   * ps_ipc_export / ps_ipc_open: CUDA IPC handles for any device pointer
//     (allocation base + offset), so torch-allocated buffers can be mapped
//     by the other ranks' processes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "ps_common.cuh"

namespace ps {
namespace {

template <int SIDE>
__global__ void __launch_bounds__(256)
    export_peer_kernel(const uint32_t *src, int64_t src_w, int64_t ppr, const int64_t *entries,
                       const int64_t *entry_count, int64_t probe_begin, int64_t probe_end,
                       int64_t slots_per_row, uint32_t *dst, int64_t dst_w, uint32_t *last_sent,
                       int64_t *last_sent_seq, int64_t current_seq, const int64_t *seq_dev) {
    constexpr int CORE = SIDE - 2;
    const int64_t count = *entry_count;
    if (seq_dev) current_seq = *seq_dev;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e = warp; e < count; e += nwarps) {
        const int64_t slot = entries[2 * e], p = entries[2 * e + 1];
        if (lane == 0 && last_sent_seq) last_sent_seq[p] = current_seq;  // replicated stamp
        if (p < probe_begin || p >= probe_end) continue;
        int64_t y0, x0;
        block_origin(p, ppr, SIDE, y0, x0);
        int64_t sy, sx;
        block_origin(slot, slots_per_row, CORE, sy, sx);
        warp_copy_block<SIDE>(src, src_w, y0, x0, lane, last_sent, [&](int r, int c, uint32_t v) {
            dst[(sy + r) * dst_w + sx + c] = v;  // encoder's atlas, maybe remote
        });
    }
}

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void peer_signal_kernel(int64_t *const *flags, int n, int64_t value,
                                   const int64_t *value_dev, int64_t add) {
    const int64_t v = (value_dev ? *value_dev : value) + add;
    __threadfence_system();  // the stream's earlier stores (remote ones included) first
    for (int i = threadIdx.x; i < n; i += blockDim.x) st_release_sys(flags[i], v);
}

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Bounded acquire spin.  A peer that never signals (crashed rank, lost
// process) would otherwise hang every GPU inside this kernel -- inside graph
// replays too, where no host watchdog sees it.  After timeout_ns the waiter
// records (flag index + 1) in *error (host-mapped pinned memory, read by
// ps_peer_status without a synchronisation) and returns; the host raises
// PS_ERR_CUDA at its next check.
__global__ void peer_wait_kernel(const int64_t *flags, int n, int64_t value,
                                 const int64_t *value_dev, int64_t add, int32_t *error,
                                 int64_t timeout_ns) {
    const int64_t v = (value_dev ? *value_dev : value) + add;
    const uint64_t t0 = global_ns();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        uint32_t spins = 0;
        while (ld_acquire_sys(flags + i) < v) {
            __nanosleep(64);
            if (error && timeout_ns > 0 && (++spins & 1023) == 0 &&
                int64_t(global_ns() - t0) > timeout_ns) {
                atomicCAS(error, 0, i + 1);
                break;
            }
        }
    }
    __threadfence_system();
}

typedef CUresult (*GetAddressRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

GetAddressRangeFn address_range_fn() {
    static GetAddressRangeFn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        check_cuda(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
        if (!f || q != cudaDriverEntryPointSuccess) fail(PS_ERR_CUDA, "cuMemGetAddressRange unavailable");
        return reinterpret_cast<GetAddressRangeFn>(f);
    }();
    return fn;
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

int ps_export_tiles_peer(int kind, const void *source, int64_t probe_count,
                         int64_t probes_per_row, const int64_t *entries,
                         const int64_t *entry_count, int64_t max_entries, int64_t probe_begin,
                         int64_t probe_end, int64_t slots_per_row, void *dst_update_texels,
                         int64_t dst_row_stride, void *last_sent, int64_t *last_sent_seq,
                         int64_t current_seq, const int64_t *current_seq_dev, void *stream) {
    PS_ABI_BEGIN
    if (kind != PS_KIND_COLOR && kind != PS_KIND_VISIBILITY) fail(PS_ERR_VALUE, "bad kind");
    if (probes_per_row < 1 || slots_per_row < 1) fail(PS_ERR_LAYOUT, "bad atlas layout");
    if (!dst_update_texels) fail(PS_ERR_VALUE, "destination update atlas missing");
    if (probe_begin < 0 || probe_end > probe_count || probe_begin > probe_end)
        fail(PS_ERR_INDEX, "probe range outside the volume");
    auto s = as_stream(stream);
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(max_entries, 8), 4096)));
    if (kind == PS_KIND_COLOR)
        export_peer_kernel<10><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), probes_per_row * 10, probes_per_row, entries,
            entry_count, probe_begin, probe_end, slots_per_row,
            static_cast<uint32_t *>(dst_update_texels), dst_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    else
        export_peer_kernel<18><<<blocks, 256, 0, s>>>(
            static_cast<const uint32_t *>(source), probes_per_row * 18, probes_per_row, entries,
            entry_count, probe_begin, probe_end, slots_per_row,
            static_cast<uint32_t *>(dst_update_texels), dst_row_stride,
            static_cast<uint32_t *>(last_sent), last_sent_seq, current_seq, current_seq_dev);
    check_launch("export_peer_kernel");
    PS_ABI_END
}

int ps_peer_signal(int64_t *const *flags, int32_t nflags, int64_t value,
                   const int64_t *value_dev, int64_t add, void *stream) {
    PS_ABI_BEGIN
    if (!flags || nflags < 1) fail(PS_ERR_VALUE, "no flags to signal");
    peer_signal_kernel<<<1, 32, 0, as_stream(stream)>>>(flags, nflags, value, value_dev, add);
    check_launch("peer_signal_kernel");
    PS_ABI_END
}

int ps_peer_wait(const int64_t *flags, int32_t nflags, int64_t value, const int64_t *value_dev,
                 int64_t add, int32_t *error, int64_t timeout_ns, void *stream) {
    PS_ABI_BEGIN
    if (!flags || nflags < 1) fail(PS_ERR_VALUE, "no flags to wait on");
    peer_wait_kernel<<<1, 32, 0, as_stream(stream)>>>(flags, nflags, value, value_dev, add, error,
                                                      timeout_ns);
    check_launch("peer_wait_kernel");
    PS_ABI_END
}

int ps_peer_status(const int32_t *error) {
    PS_ABI_BEGIN
    if (!error) fail(PS_ERR_VALUE, "null error word");
    const int32_t e = *reinterpret_cast<const volatile int32_t *>(error);
    if (e != 0)
        fail(PS_ERR_CUDA, "peer exchange timed out: rank flag " + std::to_string(e - 1) +
                              " was never signalled (a peer rank stopped or crashed)");
    PS_ABI_END
}

int ps_ipc_export(const void *ptr, uint8_t *handle, int64_t *offset) {
    PS_ABI_BEGIN
    if (!ptr || !handle || !offset) fail(PS_ERR_VALUE, "null argument");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (address_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        fail(PS_ERR_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof(h));
    *offset = int64_t(reinterpret_cast<CUdeviceptr>(ptr) - base);
    PS_ABI_END
}

size_t ps_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int ps_ipc_open(const uint8_t *handle, int64_t offset, void **ptr) {
    PS_ABI_BEGIN
    if (!handle || !ptr) fail(PS_ERR_VALUE, "null argument");
    // one mapping per allocation and process (CUDA refuses to map a handle twice)
    static std::mutex mu;
    static std::map<std::string, void *> opened;
    std::lock_guard<std::mutex> lock(mu);
    const std::string key(reinterpret_cast<const char *>(handle), sizeof(cudaIpcMemHandle_t));
    auto it = opened.find(key);
    void *base = nullptr;
    if (it != opened.end()) {
        base = it->second;
    } else {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        check_cuda(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess),
                   "cudaIpcOpenMemHandle");
        opened[key] = base;
    }
    *ptr = static_cast<char *>(base) + offset;
    PS_ABI_END
}

}  // extern "C"
