// CPU-tier swap engine: moves KV pages between the HBM page pools and a pinned host tier,
// layer-pipelined and ordered the way the reference's timeline model prescribes
// (/root/reference/proj/src/swap_engine.cpp:21-53):
//   * swap-in is issued layer by layer (layer l of every chunk before layer l+1); an event per
//     layer lets the compute stream start layer l's attention as soon as its pages landed
//     (the LayerDependencyAuditor rule of src/event_log.cpp:90-118);
//   * swap-out (D2H) follows the step's swap-ins, as in the reference's order
//     (schedule_swap_out_start, :50-53), but on its own stream: the next
//     step's swap-ins and attention do not queue behind it (pb_tier_set_policy can put it on
//     the copy stream, or run it concurrently with the swap-ins);
//   * swap-in is a batched H2D into staging plus a scatter kernel per layer block, or (policy
//     PB_SWAP_IN_ZERO_COPY) one zero-copy kernel per layer reading the mapped pinned tier;
//   * the swap-out GATHER (device pages -> contiguous staging) runs first, on the compute
//     stream, so device slots vacated by swap-out can be refilled in the same step by restore /
//     rematerialize / append (the reference reuses them LIFO, src/paged_kv_cache.cpp:28-37)
//     without a read-after-write hazard; the swap-in scatter waits for that gather;
//   * across steps the D2H is decoupled from the copy stream: a step's swap-ins wait for the
//     newest in-flight D2H (of any earlier step) that writes a host slot they read, and a D2H
//     waits for the previous step's swap-ins (a host slot freed by restore may be reused);
//   * within a step, a chunk evicted and restored again is restored device-to-device from
//     the swap-out staging (its host copy is dead and its D2H skipped), and an out-move whose
//     host slot a later out-move reuses is dropped (include/pensieve_b200.h has the rules).
// Host tier layout: [host_slot][layer][K|V][page] — one chunk's bytes for all layers are
// contiguous (= ModelConfig::chunk_bytes per worker, src/model_config.cpp:36-40), so a
// swap-out is one D2H per chunk; a swap-in reads one (K,V) block per chunk per layer.
#include "pb_common.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <deque>
#include <memory>
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

int n_sms() { return device_sms(); }

// One cudaMemcpyAsync per copy, in list order on one stream.  (The driver's batched-copy
// entry point faulted the GPU on this driver/part, so it is not used.)
void copy_batch(std::vector<void*>& dst, std::vector<void*>& src, std::vector<size_t>& sizes, cudaStream_t st) {
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
    // D2H copies not yet known complete: the host slots each one writes (sorted) and the event
    // recorded after it.  Every D2H runs on one stream (the tier's own, or the copy stream),
    // so waiting for the newest entry that writes a slot also covers the older ones.
    struct InFlight {
        cudaEvent_t ev;
        std::vector<int32_t> slots;
    };
    std::deque<InFlight> d2h_inflight;
    std::vector<cudaEvent_t> ev_pool;
    int par = 0;
    const uint8_t* host_dev = nullptr; // device alias of the pinned tier (zero-copy swap-in)
    cudaStream_t d2h = nullptr;    // swap-out D2H stream (PB_D2H_AFTER_SWAP_IN / _CONCURRENT)
    int swap_in = PB_SWAP_IN_STAGED, d2h_order = PB_D2H_AFTER_SWAP_IN;
    int layer_block = 1;           // staged swap-in: layers per H2D piece (larger pieces, coarser events)
    pb_event_log* log = nullptr;   // optional: stamps SWAP_IN_LAYER / SWAP_OUT
    cudaEvent_t gathered = nullptr, done = nullptr, in_done = nullptr;
    std::vector<cudaEvent_t> layer_ready;
    int64_t chunk_bytes() const { return static_cast<int64_t>(n_layer) * 2 * page_bytes; }

    cudaEvent_t take_event() {
        if (ev_pool.empty()) {
            cudaEvent_t e = nullptr;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    void retire_completed() { // non-blocking: drop the D2H entries whose event has fired
        while (!d2h_inflight.empty()) {
            const cudaError_t q = cudaEventQuery(d2h_inflight.front().ev);
            if (q == cudaErrorNotReady) {
                cudaGetLastError(); // not an error: do not leave it for the next launch check
                break;
            }
            if (q != cudaSuccess) cuda_check(q, "swap-out completion query");
            ev_pool.push_back(d2h_inflight.front().ev);
            d2h_inflight.pop_front();
        }
    }
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
        void* hd = nullptr;
        if (cudaHostGetDevicePointer(&hd, T->host, 0) == cudaSuccess) T->host_dev = static_cast<const uint8_t*>(hd);
        else cudaGetLastError();
        // default policy (measured, profiles/): staged swap-in in 8-layer pieces; D2H on the
        // tier's stream after the step's swap-ins, so the swap-ins (on the attention's
        // critical path) get the link alone and the D2H overlaps the following steps
        T->layer_block = std::max(1, std::min(n_layer, kDefaultLayerBlock));
        cuda_check(cudaStreamCreateWithFlags(&T->d2h, cudaStreamNonBlocking), "d2h stream");
        cuda_check(cudaEventCreateWithFlags(&T->gathered, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&T->in_done, cudaEventDisableTiming), "event");
        cuda_check(cudaEventCreateWithFlags(&T->done, cudaEventDisableTiming), "event");
        T->layer_ready.resize(static_cast<size_t>(n_layer));
        for (auto& e : T->layer_ready) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        *out = T.release();
    });
}

pb_status pb_tier_set_policy(pb_kv_tier* T, int32_t swap_in, int32_t d2h, int32_t layers_per_piece) {
    return guarded([&] {
        if (!T) fail(PB_ERR_ERROR, "null tier");
        if (swap_in != PB_SWAP_IN_STAGED && swap_in != PB_SWAP_IN_ZERO_COPY)
            fail(PB_ERR_CONFIG, "unknown swap-in method");
        if (swap_in == PB_SWAP_IN_ZERO_COPY && !T->host_dev)
            fail(PB_ERR_UNSUPPORTED, "zero-copy swap-in needs a mapped pinned tier");
        if (d2h != PB_D2H_ON_COPY_STREAM && d2h != PB_D2H_CONCURRENT && d2h != PB_D2H_AFTER_SWAP_IN)
            fail(PB_ERR_CONFIG, "unknown swap-out ordering");
        if (layers_per_piece < 0 || layers_per_piece > T->n_layer)
            fail(PB_ERR_CONFIG, "layers_per_piece must be in [0, n_layer]");
        // the D2H stream changes: everything issued so far must be done first
        for (int b = 0; b < 2; ++b) {
            cuda_check(cudaEventSynchronize(T->done_p[b]), "policy change");
            cuda_check(cudaEventSynchronize(T->d2h_p[b]), "policy change");
        }
        for (auto& f : T->d2h_inflight) {
            cuda_check(cudaEventSynchronize(f.ev), "policy change");
            T->ev_pool.push_back(f.ev);
        }
        T->d2h_inflight.clear();
        T->swap_in = swap_in;
        T->d2h_order = d2h;
        if (layers_per_piece > 0) T->layer_block = layers_per_piece;
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
    for (auto& f : T->d2h_inflight) {
        cudaEventSynchronize(f.ev);
        cudaEventDestroy(f.ev);
    }
    for (auto e : T->ev_pool) cudaEventDestroy(e);
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
        // ---- classify the step's moves (evictions precede restores within a step) ----
        // from_stage[j] = out-move whose staged bytes restore in-move j (same chunk evicted to
        // the host slot it is restored from, this step), else -1
        std::vector<int64_t> from_stage(static_cast<size_t>(n_in), -1);
        std::vector<char> live(static_cast<size_t>(n_out), 1);
        for (int64_t j = 0; j < n_in; ++j)
            for (int64_t i = n_out - 1; i >= 0; --i)
                if (out_moves[i].chunk == in_moves[j].chunk && out_moves[i].dst_slot == in_moves[j].src_slot) {
                    from_stage[static_cast<size_t>(j)] = i;
                    live[static_cast<size_t>(i)] = 0; // host copy dead: restore freed the slot
                    break;
                }
        {
            // a later out-move to the same host slot means the earlier chunk left that slot
            // (dropped from the host) in between: only the last write is live
            std::vector<std::pair<int32_t, int64_t>> by_slot;
            for (int64_t i = 0; i < n_out; ++i) by_slot.push_back({out_moves[i].dst_slot, i});
            std::sort(by_slot.begin(), by_slot.end());
            for (size_t a = 0; a + 1 < by_slot.size(); ++a)
                if (by_slot[a].first == by_slot[a + 1].first) live[static_cast<size_t>(by_slot[a].second)] = 0;
        }
        int64_t n_host_in = 0, n_live_out = 0;
        for (int64_t j = 0; j < n_in; ++j) n_host_in += from_stage[static_cast<size_t>(j)] < 0;
        for (int64_t i = 0; i < n_out; ++i) n_live_out += live[static_cast<size_t>(i)];
        cudaStream_t cs = as_stream(compute_stream), xs = as_stream(copy_stream);
        // this step's buffers were last used two steps ago: only that step must be done
        const int par = T->par;
        T->par ^= 1;
        cuda_check(cudaEventSynchronize(T->done_p[par]), "swap step ordering");
        T->retire_completed();
        int32_t* h_slots = T->h_slots[par];
        int32_t* d_slots = T->d_slots[par];
        uint8_t* stage_out = T->stage_out[par];
        uint8_t* stage_in = T->stage_in[par];
        for (int64_t i = 0; i < n_out; ++i) h_slots[i] = out_moves[i].src_slot;
        for (int64_t i = 0; i < n_in; ++i) h_slots[T->max_chunks + i] = in_moves[i].dst_slot;
        for (int64_t i = 0; i < n_in; ++i) h_slots[2 * T->max_chunks + i] = in_moves[i].src_slot;
        cuda_check(cudaMemcpyAsync(d_slots, h_slots, sizeof(int32_t) * 3 * T->max_chunks, cudaMemcpyHostToDevice, cs),
                   "slot upload");
        // RAW across steps: a swap-in from the host reads a slot some earlier step's D2H may
        // still be writing -> wait for the newest such D2H
        cudaEvent_t raw_ev = nullptr;
        for (auto it = T->d2h_inflight.rbegin(); it != T->d2h_inflight.rend() && !raw_ev; ++it)
            for (int64_t j = 0; j < n_in; ++j)
                if (from_stage[static_cast<size_t>(j)] < 0 &&
                    std::binary_search(it->slots.begin(), it->slots.end(), in_moves[j].src_slot)) {
                    raw_ev = it->ev;
                    break;
                }
        // WAR within the step: a live swap-out overwrites a host slot a restore of another
        // chunk reads (restore frees host slots at once) -> that D2H follows the swap-ins
        bool war = false;
        for (int64_t i = 0; i < n_out && !war; ++i) {
            if (!live[static_cast<size_t>(i)]) continue;
            for (int64_t j = 0; j < n_in; ++j)
                if (from_stage[static_cast<size_t>(j)] < 0 && out_moves[i].dst_slot == in_moves[j].src_slot) {
                    war = true;
                    break;
                }
        }
        const int64_t pb = T->page_bytes;
        auto* kp = static_cast<uint8_t*>(k_pool);
        auto* vp = static_cast<uint8_t*>(v_pool);
        // 1. swap-out gather on the compute stream, before any same-step write to those slots;
        // stage_out[par] is free once the D2H of two steps ago is done, and the device slots it
        // reads may have been filled by the previous step's swap-ins (stream waits: the host
        // never blocks on a D2H that may still run under later steps' attention)
        if (n_out > 0) {
            cuda_check(cudaStreamWaitEvent(cs, T->d2h_p[par], 0), "stream wait");
            cuda_check(cudaStreamWaitEvent(cs, T->done_p[par ^ 1], 0), "stream wait");
            const int64_t jobs = n_out * T->n_layer * 2;
            const int grid = static_cast<int>(std::min<int64_t>(jobs, n_sms() * 8));
            swap_gather_kernel<<<grid, 256, 0, cs>>>(kp, vp, layer_stride, pb, d_slots, static_cast<int32_t>(n_out),
                                                     T->n_layer, stage_out);
            cuda_check(cudaGetLastError(), "swap gather");
            count_launch();
        }
        cuda_check(cudaEventRecord(T->gathered, cs), "event record");
        cuda_check(cudaStreamWaitEvent(xs, T->gathered, 0), "stream wait");
        if (raw_ev) cuda_check(cudaStreamWaitEvent(xs, raw_ev, 0), "stream wait");
        // 2. swap-in, layer by layer: H2D (batched) into staging, scatter, per-layer event;
        // chunks restored from this step's own swap-out come device-to-device from stage_out
        const bool zc = T->swap_in == PB_SWAP_IN_ZERO_COPY && n_host_in == n_in;
        std::vector<void*> dst, src;
        std::vector<size_t> sz;
        for (int32_t l = 0; l < T->n_layer; ++l) {
            if (n_in > 0 && zc) {
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
                const int64_t layer_off = static_cast<int64_t>(l) * 2 * pb;
                for (int64_t i = 0; i < n_in; ++i) {
                    const int64_t o = from_stage[static_cast<size_t>(i)];
                    if (o >= 0) continue;
                    dst.push_back(stage_b + i * nl * 2 * pb);
                    src.push_back(T->host + static_cast<int64_t>(in_moves[i].src_slot) * T->chunk_bytes() + layer_off);
                    sz.push_back(static_cast<size_t>(nl * 2 * pb));
                }
                copy_batch(dst, src, sz, xs);
                for (int64_t i = 0; i < n_in; ++i) {
                    const int64_t o = from_stage[static_cast<size_t>(i)];
                    if (o < 0) continue;
                    cuda_check(cudaMemcpyAsync(stage_b + i * nl * 2 * pb, stage_out + o * T->chunk_bytes() + layer_off,
                                               static_cast<size_t>(nl * 2 * pb), cudaMemcpyDeviceToDevice, xs),
                               "swap-in from staging");
                }
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
        // 3. swap-out D2H of the live out-moves.  Every D2H of the tier runs on one stream (the
        // tier's own, or the copy stream for PB_D2H_ON_COPY_STREAM) so they complete in order.
        cudaStream_t os = xs;
        if (T->d2h_order != PB_D2H_ON_COPY_STREAM) {
            os = T->d2h;
            cuda_check(cudaStreamWaitEvent(os, T->gathered, 0), "stream wait");
            if (n_in > 0 && (T->d2h_order == PB_D2H_AFTER_SWAP_IN || war)) {
                cuda_check(cudaEventRecord(T->in_done, xs), "event record");
                cuda_check(cudaStreamWaitEvent(os, T->in_done, 0), "stream wait");
            }
            // cross-step WAR: the previous step's swap-ins may still read a host slot this
            // D2H reuses (restore frees host slots at once)
            cuda_check(cudaStreamWaitEvent(os, T->done_p[par ^ 1], 0), "stream wait");
        }
        if (n_live_out > 0) {
            dst.clear();
            src.clear();
            sz.clear();
            std::vector<int32_t> slots;
            for (int64_t i = 0; i < n_out; ++i) {
                if (!live[static_cast<size_t>(i)]) continue;
                dst.push_back(T->host + static_cast<int64_t>(out_moves[i].dst_slot) * T->chunk_bytes());
                src.push_back(stage_out + i * T->chunk_bytes());
                sz.push_back(static_cast<size_t>(T->chunk_bytes()));
                slots.push_back(out_moves[i].dst_slot);
            }
            copy_batch(dst, src, sz, os);
            if (T->log) {
                const pb_status r = pb_evlog_mark(T->log, PB_EV_SWAP_OUT, -1, -1, os);
                if (r != PB_OK) fail(r, "swap-out stamp");
            }
            std::sort(slots.begin(), slots.end());
            cudaEvent_t e = T->take_event();
            cuda_check(cudaEventRecord(e, os), "event record");
            T->d2h_inflight.push_back({e, std::move(slots)});
        }
        cuda_check(cudaEventRecord(T->d2h_p[par], os), "event record");
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
        for (auto& f : T->d2h_inflight) cuda_check(cudaEventSynchronize(f.ev), "swap sync");
        T->retire_completed();
    });
}

} // extern "C"
