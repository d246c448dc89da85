// CPU-tier swap engine: moves KV pages between the HBM page pools and a pinned host tier,
// layer-pipelined and ordered the way the reference's timeline model prescribes
// (/root/reference/proj/src/swap_engine.cpp:21-53):
//   * swap-in is issued layer by layer (layer l of every chunk before layer l+1); an event per
//     layer lets the compute stream start layer l's attention as soon as its pages landed
//     (the LayerDependencyAuditor rule of src/event_log.cpp:90-118);
//   * swap-out (D2H) follows the step's swap-ins, as in the reference's order
//     (schedule_swap_out_start, :50-53), but on its own stream: the next
//     step's swap-ins and attention do not queue behind it (PB_SWAP_DUPLEX=0 puts it on the
//     copy stream, =1 runs it concurrently with the swap-ins);
//   * swap-in is a batched H2D into staging plus a scatter kernel per layer, or with
//     PB_SWAP_IN=zc one zero-copy kernel per layer reading the mapped pinned tier;
//   * the swap-out GATHER (device pages -> contiguous staging) runs first, on the compute
//     stream, so device slots vacated by swap-out can be refilled in the same step by restore /
//     rematerialize / append (the reference reuses them LIFO, src/paged_kv_cache.cpp:28-37)
//     without a read-after-write hazard; the swap-in scatter waits for that gather;
//   * across steps the D2H is decoupled from the copy stream: a step's swap-ins wait for the
//     previous step's D2H only when they read a host slot it writes, and a D2H waits for the
//     previous step's swap-ins (a host slot freed by restore may be reused at once).
// Host tier layout: [host_slot][layer][K|V][page] — one chunk's bytes for all layers are
// contiguous (= ModelConfig::chunk_bytes per worker, src/model_config.cpp:36-40), so a
// swap-out is one D2H per chunk; a swap-in reads one (K,V) block per chunk per layer.
#include "pb_common.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <cstdlib>
#include <string>
#include <vector>

namespace pb {
namespace {

constexpr int kDefaultLayerBlock = 8; // swap-in H2D pieces of 8 layers (measured best of 1, 2, 4, 8, 40)

__global__ void __launch_bounds__(256) swap_gather_kernel(const uint8_t* __restrict__ kpool,
                                                          const uint8_t* __restrict__ vpool, int64_t layer_stride,
                                                          int64_t page_bytes, const int32_t* __restrict__ slots,
                                                          int32_t n, int32_t n_layer, uint8_t* __restrict__ stage) {
    // job = (chunk i, layer l, K|V); staging[((i*L + l)*2 + kv) * page]
    const int64_t jobs = static_cast<int64_t>(n) * n_layer * 2;
    const int64_t vecs = page_bytes / 16;
    for (int64_t job = blockIdx.x; job < jobs; job += gridDim.x) {
        const int kv = static_cast<int>(job & 1);
        const int64_t il = job >> 1;
        const int64_t i = il / n_layer, l = il % n_layer;
        const int4* src = reinterpret_cast<const int4*>((kv ? vpool : kpool) + l * layer_stride +
                                                        static_cast<int64_t>(slots[i]) * page_bytes);
        int4* dst = reinterpret_cast<int4*>(stage + job * page_bytes);
        for (int64_t v = threadIdx.x; v < vecs; v += blockDim.x) __stcs(dst + v, __ldcs(src + v));
    }
}

// Swap-in straight from the pinned host tier (zero-copy, mapped memory): one launch per layer
// reads every swapped-in chunk's K and V page of that layer over PCIe / C2C and writes it into
// the pool, with no staging buffer and no per-piece copy calls.  Four 16-B loads in flight per
// thread keep enough requests outstanding to fill the link.
__global__ void __launch_bounds__(256) swap_in_zc_layer_kernel(const uint8_t* __restrict__ host, int64_t chunk_bytes,
                                                               int64_t layer_off, int64_t page_bytes,
                                                               const int32_t* __restrict__ src_slots,
                                                               const int32_t* __restrict__ dst_slots, int32_t n,
                                                               uint8_t* __restrict__ kpool_l,
                                                               uint8_t* __restrict__ vpool_l) {
    const int64_t vecs = page_bytes / 16;
    const int64_t total = static_cast<int64_t>(n) * 2 * vecs;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    auto addr = [&](int64_t x, const int4*& src, int4*& dst) {
        const int64_t job = x / vecs, e = x - job * vecs;
        const int kv = static_cast<int>(job & 1);
        const int64_t i = job >> 1;
        src = reinterpret_cast<const int4*>(host + static_cast<int64_t>(src_slots[i]) * chunk_bytes + layer_off +
                                            kv * page_bytes) + e;
        dst = reinterpret_cast<int4*>((kv ? vpool_l : kpool_l) + static_cast<int64_t>(dst_slots[i]) * page_bytes) + e;
    };
    for (; v + 3 * stride < total; v += 4 * stride) {
        const int4 *s0, *s1, *s2, *s3;
        int4 *d0, *d1, *d2, *d3;
        addr(v, s0, d0);
        addr(v + stride, s1, d1);
        addr(v + 2 * stride, s2, d2);
        addr(v + 3 * stride, s3, d3);
        const int4 a = __ldcv(s0), b = __ldcv(s1), c = __ldcv(s2), d = __ldcv(s3);
        *d0 = a;
        *d1 = b;
        *d2 = c;
        *d3 = d;
    }
    for (; v < total; v += stride) {
        const int4* s0;
        int4* d0;
        addr(v, s0, d0);
        *d0 = __ldcv(s0);
    }
}

// Scatter of one block of nl layers: staging [chunk i][layer ll][K|V][page] -> the pools of
// layers layer0 .. layer0+nl-1.
__global__ void __launch_bounds__(256) swap_scatter_block_kernel(const uint8_t* __restrict__ stage,
                                                                 uint8_t* __restrict__ kpool, uint8_t* __restrict__ vpool,
                                                                 int64_t layer_stride, int32_t layer0, int32_t nl,
                                                                 int64_t page_bytes, const int32_t* __restrict__ slots,
                                                                 int32_t n) {
    const int64_t jobs = static_cast<int64_t>(n) * nl * 2;
    const int64_t vecs = page_bytes / 16;
    for (int64_t job = blockIdx.x; job < jobs; job += gridDim.x) {
        const int kv = static_cast<int>(job & 1);
        const int64_t il = job >> 1;
        const int64_t i = il / nl, ll = il % nl;
        const int4* src = reinterpret_cast<const int4*>(stage + job * page_bytes);
        int4* dst = reinterpret_cast<int4*>((kv ? vpool : kpool) + (layer0 + ll) * layer_stride +
                                            static_cast<int64_t>(slots[i]) * page_bytes);
        for (int64_t v = threadIdx.x; v < vecs; v += blockDim.x) __stcs(dst + v, __ldcs(src + v));
    }
}

int n_sms() {
    static int s = 0;
    if (!s) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        if (s <= 0) s = 148;
    }
    return s;
}

// Batched copies (one driver call per batch, cudaMemcpyBatchAsync); per-copy fallback if the
// runtime refuses the batch.
void copy_batch(std::vector<void*>& dst, std::vector<void*>& src, std::vector<size_t>& sizes, cudaStream_t st) {
    if (dst.empty()) return;
    static const int use_batch = [] { // profiling knob: 0 = one cudaMemcpyAsync per piece
        const char* e = std::getenv("PB_SWAP_BATCH");
        return e ? std::atoi(e) : 1;
    }();
    if (!use_batch) {
        for (size_t i = 0; i < dst.size(); ++i)
            cuda_check(cudaMemcpyAsync(dst[i], src[i], sizes[i], cudaMemcpyDefault, st), "swap copy");
        return;
    }
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    size_t attr_idx = 0, fail_idx = 0;
    cudaError_t e = cudaMemcpyBatchAsync(dst.data(), src.data(), sizes.data(), dst.size(), &attr, &attr_idx, 1,
                                         &fail_idx, st);
    if (e == cudaSuccess) return;
    cudaGetLastError();
    for (size_t i = 0; i < dst.size(); ++i)
        cuda_check(cudaMemcpyAsync(dst[i], src[i], sizes[i], cudaMemcpyDefault, st), "swap copy");
}

} // namespace
} // namespace pb

using namespace pb;

struct pb_kv_tier {
    int32_t n_layer = 0, host_slots = 0, max_chunks = 0;
    int64_t page_bytes = 0;
    uint8_t* host = nullptr;       // pinned [host_slot][layer][K|V][page]
    // per-step buffers, double-buffered by step parity so step s+1 can be issued while step
    // s's transfers (the swap-out D2H above all) are still running
    uint8_t* stage_out[2] = {};    // device [chunk][layer][K|V][page]
    uint8_t* stage_in[2] = {};     // device [layer block][chunk][layers][K|V][page]
    int32_t* d_slots[2] = {};      // device: [out src slots | in dst slots | in host src slots]
    int32_t* h_slots[2] = {};      // pinned staging for the slot lists
    cudaEvent_t done_p[2] = {};    // swap-ins of the step with this parity done (copy stream)
    cudaEvent_t d2h_p[2] = {};     // swap-out D2H of the step with this parity done
    cudaEvent_t d2h_prev = nullptr; // last issued swap-out D2H (host-slot RAW for swap-ins)
    std::vector<int32_t> prev_out_dst; // host slots the previous step's D2H writes (sorted)
    int par = 0;
    const uint8_t* host_dev = nullptr; // device alias of the pinned tier (zero-copy swap-in)
    cudaStream_t d2h = nullptr;    // duplex mode: swap-out D2H on its own stream
    int mode_zc = 0, mode_duplex = 0;
    int layer_block = 1;           // staged swap-in: layers per H2D piece (larger pieces, coarser events)
    pb_event_log* log = nullptr;   // optional: stamps SWAP_IN_LAYER / SWAP_OUT
    cudaEvent_t gathered = nullptr, done = nullptr, in_done = nullptr;
    std::vector<cudaEvent_t> layer_ready;
    bool any_in = false;
    int64_t chunk_bytes() const { return static_cast<int64_t>(n_layer) * 2 * page_bytes; }
};

extern "C" {

pb_status pb_tier_create(int32_t n_layer, int32_t host_slots, int64_t page_bytes, int32_t max_chunks_per_step,
                         pb_kv_tier** out) {
    return guarded([&] {
        if (!out) fail(PB_ERR_ERROR, "null out");
        *out = nullptr;
        if (n_layer < 1 || host_slots < 0 || page_bytes <= 0 || page_bytes % 16 || max_chunks_per_step < 1)
            fail(PB_ERR_CONFIG, "bad tier geometry (page_bytes must be a positive multiple of 16)");
        auto T = std::make_unique<pb_kv_tier>();
        T->n_layer = n_layer;
        T->host_slots = host_slots;
        T->page_bytes = page_bytes;
        T->max_chunks = max_chunks_per_step;
        const size_t host_bytes = static_cast<size_t>(std::max(1, host_slots)) * T->chunk_bytes();
        if (cudaHostAlloc(reinterpret_cast<void**>(&T->host), host_bytes, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            fail(PB_ERR_INSUFFICIENT_HOST_MEMORY, "pinned host tier allocation failed");
        }
        const size_t stage_bytes = static_cast<size_t>(max_chunks_per_step) * T->chunk_bytes();
        for (int b = 0; b < 2; ++b) {
            if (cudaMalloc(&T->stage_out[b], stage_bytes) != cudaSuccess ||
                cudaMalloc(&T->stage_in[b], stage_bytes) != cudaSuccess) {
                cudaGetLastError();
                fail(PB_ERR_INSUFFICIENT_DEVICE_MEMORY, "swap staging allocation failed");
            }
            cuda_check(cudaMalloc(&T->d_slots[b], sizeof(int32_t) * 3 * max_chunks_per_step), "cudaMalloc(slots)");
            cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&T->h_slots[b]), sizeof(int32_t) * 3 * max_chunks_per_step,
                                     cudaHostAllocPortable),
                       "cudaHostAlloc(slots)");
            cuda_check(cudaEventCreateWithFlags(&T->done_p[b], cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&T->d2h_p[b], cudaEventDisableTiming), "event");
        }
        cuda_check(cudaEventCreateWithFlags(&T->d2h_prev, cudaEventDisableTiming), "event");
        void* hd = nullptr;
        if (cudaHostGetDevicePointer(&hd, T->host, 0) == cudaSuccess) T->host_dev = static_cast<const uint8_t*>(hd);
        else cudaGetLastError();
        // transfer policy: zero-copy swap-in (default) or staged H2D + scatter; swap-out D2H
        // behind the swap-ins (reference order, default) or on its own stream (duplex)
        const char* m = std::getenv("PB_SWAP_IN");
        T->mode_zc = T->host_dev && m && std::string(m) == "zc"; // staged measured faster
        const char* dx = std::getenv("PB_SWAP_DUPLEX");
        // 0: D2H queued behind the swap-ins on the copy stream (the reference's order);
        // 1: D2H concurrent with the swap-ins on its own stream; 2 (default): on its own stream
        // after this step's swap-ins, so the swap-ins (on the attention's critical path) get
        // the link alone and the D2H overlaps the following steps (measured, profiles/)
        T->mode_duplex = dx ? std::atoi(dx) : 2;
        const char* lb = std::getenv("PB_SWAP_LB");
        T->layer_block = std::max(1, std::min(n_layer, lb ? std::atoi(lb) : kDefaultLayerBlock));
        cuda_check(cudaStreamCreateWithFlags(&T->d2h, cudaStreamNonBlocking), "d2h stream");
        cuda_check(cudaEventCreateWithFlags(&T->gathered, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&T->in_done, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&T->done, cudaEventDisableTiming), "event");
        T->layer_ready.resize(static_cast<size_t>(n_layer));
        for (auto& e : T->layer_ready) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        *out = T.release();
    });
}

void pb_tier_destroy(pb_kv_tier* T) {
    if (!T) return;
    if (T->done) cudaEventSynchronize(T->done);
    for (int b = 0; b < 2; ++b) {
        if (T->done_p[b]) {
            cudaEventSynchronize(T->done_p[b]);
            cudaEventDestroy(T->done_p[b]);
        }
        if (T->d2h_p[b]) {
            cudaEventSynchronize(T->d2h_p[b]);
            cudaEventDestroy(T->d2h_p[b]);
        }
        cudaFree(T->stage_out[b]);
        cudaFree(T->stage_in[b]);
        cudaFree(T->d_slots[b]);
        cudaFreeHost(T->h_slots[b]);
    }
    if (T->d2h_prev) cudaEventDestroy(T->d2h_prev);
    cudaFreeHost(T->host);
    if (T->d2h) {
        cudaStreamSynchronize(T->d2h);
        cudaStreamDestroy(T->d2h);
    }
    if (T->gathered) cudaEventDestroy(T->gathered);
    if (T->in_done) cudaEventDestroy(T->in_done);
    if (T->done) cudaEventDestroy(T->done);
    for (auto e : T->layer_ready) cudaEventDestroy(e);
    delete T;
}

void* pb_tier_host_base(pb_kv_tier* T) { return T ? T->host : nullptr; }

int64_t pb_tier_chunk_bytes(const pb_kv_tier* T) { return T ? T->chunk_bytes() : 0; }

pb_status pb_swap_step(pb_kv_tier* T, void* k_pool, void* v_pool, int64_t layer_stride, const pb_slot_move* out_moves,
                       int64_t n_out, const pb_slot_move* in_moves, int64_t n_in, void* compute_stream,
                       void* copy_stream) {
    return guarded([&] {
        if (!T) fail(PB_ERR_ERROR, "null tier");
        if (n_out < 0 || n_in < 0 || n_out > T->max_chunks || n_in > T->max_chunks)
            fail(PB_ERR_DIMENSION_MISMATCH, "swap batch exceeds the tier's max_chunks_per_step");
        for (int64_t i = 0; i < n_out; ++i)
            if (out_moves[i].src_slot < 0 || out_moves[i].dst_slot < 0 || out_moves[i].dst_slot >= T->host_slots)
                fail(PB_ERR_ERROR, "swap-out move needs a device source and a host destination slot");
        for (int64_t i = 0; i < n_in; ++i)
            if (in_moves[i].src_slot < 0 || in_moves[i].src_slot >= T->host_slots || in_moves[i].dst_slot < 0)
                fail(PB_ERR_ERROR, "swap-in move needs a host source and a device destination slot");
        cudaStream_t cs = as_stream(compute_stream), xs = as_stream(copy_stream);
        // this step's buffers were last used two steps ago: only that step must be done
        const int par = T->par;
        T->par ^= 1;
        cuda_check(cudaEventSynchronize(T->done_p[par]), "swap step ordering");
        int32_t* h_slots = T->h_slots[par];
        int32_t* d_slots = T->d_slots[par];
        uint8_t* stage_out = T->stage_out[par];
        uint8_t* stage_in = T->stage_in[par];
        for (int64_t i = 0; i < n_out; ++i) h_slots[i] = out_moves[i].src_slot;
        for (int64_t i = 0; i < n_in; ++i) h_slots[T->max_chunks + i] = in_moves[i].dst_slot;
        for (int64_t i = 0; i < n_in; ++i) h_slots[2 * T->max_chunks + i] = in_moves[i].src_slot;
        cuda_check(cudaMemcpyAsync(d_slots, h_slots, sizeof(int32_t) * 3 * T->max_chunks, cudaMemcpyHostToDevice, cs),
                   "slot upload");
        // host-slot hazards: a swap-in may read a host slot the previous step's swap-out writes
        // (RAW: then the swap-ins wait for that D2H; older steps' D2H are done, synchronised
        // above), and restore frees host slots at once, so this step's swap-out may overwrite
        // a slot one of this step's swap-ins reads (WAR: then the D2H waits for the swap-ins,
        // the reference's order, src/swap_engine.cpp:50-53)
        bool raw = false;
        for (int64_t j = 0; j < n_in && !raw; ++j)
            raw = std::binary_search(T->prev_out_dst.begin(), T->prev_out_dst.end(), in_moves[j].src_slot);
        bool war = false;
        for (int64_t i = 0; i < n_out && !war; ++i)
            for (int64_t j = 0; j < n_in; ++j)
                if (out_moves[i].dst_slot == in_moves[j].src_slot) {
                    war = true;
                    break;
                }
        const int64_t pb = T->page_bytes;
        auto* kp = static_cast<uint8_t*>(k_pool);
        auto* vp = static_cast<uint8_t*>(v_pool);
        // 1. swap-out gather on the compute stream, before any same-step write to those slots;
        // stage_out[par] is free once the D2H of two steps ago is done (a stream wait, so the
        // host does not block on a D2H that may still run under later steps' attention)
        if (n_out > 0) {
            cuda_check(cudaStreamWaitEvent(cs, T->d2h_p[par], 0), "stream wait");
            const int64_t jobs = n_out * T->n_layer * 2;
            const int grid = static_cast<int>(std::min<int64_t>(jobs, n_sms() * 8));
            swap_gather_kernel<<<grid, 256, 0, cs>>>(kp, vp, layer_stride, pb, d_slots, static_cast<int32_t>(n_out),
                                                     T->n_layer, stage_out);
            cuda_check(cudaGetLastError(), "swap gather");
            count_launch();
        }
        cuda_check(cudaEventRecord(T->gathered, cs), "event record");
        cuda_check(cudaStreamWaitEvent(xs, T->gathered, 0), "stream wait");
        if (raw) cuda_check(cudaStreamWaitEvent(xs, T->d2h_prev, 0), "stream wait");
        // 2. swap-in, layer by layer: H2D (batched) into staging, scatter, per-layer event
        T->any_in = n_in > 0;
        std::vector<void*> dst, src;
        std::vector<size_t> sz;
        for (int32_t l = 0; l < T->n_layer; ++l) {
            if (n_in > 0 && T->mode_zc) {
                const int64_t vecs = n_in * 2 * (pb / 16);
                const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((vecs + 1023) / 1024, n_sms() * 4)));
                swap_in_zc_layer_kernel<<<grid, 256, 0, xs>>>(T->host_dev, T->chunk_bytes(), static_cast<int64_t>(l) * 2 * pb,
                                                              pb, d_slots + 2 * T->max_chunks,
                                                              d_slots + T->max_chunks, static_cast<int32_t>(n_in),
                                                              kp + l * layer_stride, vp + l * layer_stride);
                cuda_check(cudaGetLastError(), "swap-in (zero-copy)");
                count_launch();
            } else if (n_in > 0 && l % T->layer_block == 0) {
                // one H2D piece per chunk for the next nl layers (contiguous in the host tier),
                // then one scatter for the block; every layer of the block is ready after it
                const int32_t nl = std::min(T->layer_block, T->n_layer - l);
                dst.clear();
                src.clear();
                sz.clear();
                uint8_t* stage_b = stage_in + static_cast<int64_t>(l) * n_in * 2 * pb;
                for (int64_t i = 0; i < n_in; ++i) {
                    dst.push_back(stage_b + i * nl * 2 * pb);
                    src.push_back(T->host + static_cast<int64_t>(in_moves[i].src_slot) * T->chunk_bytes() +
                                  static_cast<int64_t>(l) * 2 * pb);
                    sz.push_back(static_cast<size_t>(nl * 2 * pb));
                }
                copy_batch(dst, src, sz, xs);
                const int grid = static_cast<int>(std::min<int64_t>(n_in * nl * 2, n_sms() * 4));
                swap_scatter_block_kernel<<<grid, 256, 0, xs>>>(stage_b, kp, vp, layer_stride, l, nl, pb,
                                                               d_slots + T->max_chunks, static_cast<int32_t>(n_in));
                cuda_check(cudaGetLastError(), "swap scatter");
                count_launch();
            }
            if (T->log && n_in > 0) {
                const pb_status r = pb_evlog_mark(T->log, PB_EV_SWAP_IN_LAYER, l, -1, xs);
                if (r != PB_OK) fail(r, "swap-in stamp");
            }
            cuda_check(cudaEventRecord(T->layer_ready[static_cast<size_t>(l)], xs), "event record");
        }
        // 3. swap-out D2H: behind the swap-ins on the copy stream (the reference's order, no
        // duplex contention on the link), or concurrently on its own stream (duplex mode)
        cudaStream_t os = xs;
        if (T->mode_duplex && !war) {
            os = T->d2h;
            cuda_check(cudaStreamWaitEvent(os, T->gathered, 0), "stream wait");
            if (T->mode_duplex == 2 && n_in > 0) {
                cuda_check(cudaEventRecord(T->in_done, xs), "event record");
                cuda_check(cudaStreamWaitEvent(os, T->in_done, 0), "stream wait");
            }
            // cross-step WAR: the previous step's swap-ins may still read a host slot this
            // D2H reuses (restore frees host slots at once)
            cuda_check(cudaStreamWaitEvent(os, T->done_p[par ^ 1], 0), "stream wait");
        }
        if (n_out > 0) {
            dst.clear();
            src.clear();
            sz.clear();
            for (int64_t i = 0; i < n_out; ++i) {
                dst.push_back(T->host + static_cast<int64_t>(out_moves[i].dst_slot) * T->chunk_bytes());
                src.push_back(stage_out + i * T->chunk_bytes());
                sz.push_back(static_cast<size_t>(T->chunk_bytes()));
            }
            copy_batch(dst, src, sz, os);
            if (T->log) {
                const pb_status r = pb_evlog_mark(T->log, PB_EV_SWAP_OUT, -1, -1, os);
                if (r != PB_OK) fail(r, "swap-out stamp");
            }
        }
        // the D2H no longer joins the copy stream: the next step's swap-ins only wait for it
        // on a real RAW hazard
        cuda_check(cudaEventRecord(T->d2h_p[par], os), "event record");
        T->prev_out_dst.clear();
        if (n_out > 0) {
            cuda_check(cudaEventRecord(T->d2h_prev, os), "event record");
            for (int64_t i = 0; i < n_out; ++i) T->prev_out_dst.push_back(out_moves[i].dst_slot);
            std::sort(T->prev_out_dst.begin(), T->prev_out_dst.end());
        }
        cuda_check(cudaEventRecord(T->done_p[par], xs), "event record");
        cuda_check(cudaEventRecord(T->done, xs), "event record");
    });
}

pb_status pb_swap_wait_layer(pb_kv_tier* T, int32_t layer, void* compute_stream) {
    return guarded([&] {
        if (!T || layer < 0 || layer >= T->n_layer) fail(PB_ERR_DIMENSION_MISMATCH, "layer out of range");
        cuda_check(cudaStreamWaitEvent(as_stream(compute_stream), T->layer_ready[static_cast<size_t>(layer)], 0),
                   "stream wait");
    });
}

pb_status pb_tier_set_event_log(pb_kv_tier* T, pb_event_log* log) {
    return guarded([&] {
        if (!T) fail(PB_ERR_ERROR, "null tier");
        T->log = log;
    });
}

pb_status pb_swap_sync(pb_kv_tier* T) {
    return guarded([&] {
        if (!T) fail(PB_ERR_ERROR, "null tier");
        cuda_check(cudaEventSynchronize(T->done), "swap sync");
        for (int b = 0; b < 2; ++b) cuda_check(cudaEventSynchronize(T->d2h_p[b]), "swap sync");
    });
}

} // extern "C"
