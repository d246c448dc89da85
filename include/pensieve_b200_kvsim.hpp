// pensieve_b200_kvsim.hpp — drop-in adapter for the reference's C++ operator API.
//
// A kvsim translation unit that includes this header instead of calling
// kvsim::paged_multi_token_attention / kvsim::single_token_attention
// (/root/reference/proj/include/kvsim/attention.hpp:71-77) gets the same value-semantics
// signatures, the same layouts and the same exception classes, computed by the B200 C-ABI.
// The adapter is duck-typed on the reference types (RaggedQueryBatch, PagedKvStore,
// SubRequest), so it compiles without the kvsim headers too; when kvsim/errors.hpp is on the
// include path, pb_status codes are rethrown as the reference's own exceptions.
//
// dtype PB_F32 runs the fp32 validation mode (1e-5 parity); PB_BF16 rounds inputs to bf16.
#pragma once

#include "pensieve_b200.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#if __has_include("kvsim/errors.hpp")
#include "kvsim/errors.hpp"
#define PENSIEVE_B200_HAVE_KVSIM 1
#endif

namespace pensieve_b200 {

[[noreturn]] inline void raise(pb_status st) {
    const std::string msg = pb_last_error();
#ifdef PENSIEVE_B200_HAVE_KVSIM
    switch (st) {
    case PB_ERR_DIMENSION_MISMATCH: throw kvsim::DimensionMismatch(msg);
    case PB_ERR_NUMERIC: throw kvsim::NumericError(msg);
    case PB_ERR_INSUFFICIENT_DEVICE_MEMORY: throw kvsim::InsufficientDeviceMemory(msg);
    case PB_ERR_INSUFFICIENT_HOST_MEMORY: throw kvsim::InsufficientHostMemory(msg);
    case PB_ERR_INVALID_CHUNK_STATE: throw kvsim::InvalidChunkState(msg);
    case PB_ERR_UNKNOWN_CONVERSATION: throw kvsim::UnknownConversation(msg);
    case PB_ERR_CONFIG: throw kvsim::ConfigError(msg);
    case PB_ERR_NOT_ENOUGH_EVICTABLE: throw kvsim::NotEnoughEvictable(msg);
    case PB_ERR_TRACE_MISSING: throw kvsim::TraceMissing(msg);
    case PB_ERR_CANNOT_SUSPEND_ALL: throw kvsim::CannotSuspendAll(msg);
    default: throw kvsim::Error(msg);
    }
#else
    throw std::runtime_error("pb status " + std::to_string(static_cast<int>(st)) + ": " + msg);
#endif
}

template <class Batch, class Store>
std::vector<float> attention(const Batch& batch, const Store& store, bool single_token, pb_dtype dtype) {
    // check_batch's head-size agreement (attention.cpp:25-26) is a property of the two
    // objects, so it is checked here; everything else is validated by the library.
    if (!(store.n_kv_head > 0 && store.head_size == batch.head_size)) raise(PB_ERR_DIMENSION_MISMATCH);
    const std::size_t n = batch.sub_requests.size();
    std::vector<int64_t> qs(n), ql(n), cl(n), co(n), off(n + 1, 0);
    std::vector<int32_t> bt;
    for (std::size_t i = 0; i < n; ++i) {
        const auto& s = batch.sub_requests[i];
        qs[i] = s.query_start;
        ql[i] = s.query_len;
        cl[i] = s.context_len;
        co[i] = s.causal_offset;
        bt.insert(bt.end(), s.block_table.begin(), s.block_table.end());
        off[i + 1] = static_cast<int64_t>(bt.size());
    }
    if (bt.empty()) bt.push_back(0);
    const pb_attn_shape shape{batch.n_head, store.n_kv_head, batch.head_size, store.chunk_size, store.n_slots,
                              static_cast<int32_t>(dtype), batch.scale};
    const int64_t total = static_cast<int64_t>(batch.total_tokens());
    std::vector<float> out(batch.q.size(), 0.0f);
    const pb_status st =
        (single_token ? pb_single_token_attention : pb_paged_multi_token_attention)(
            &shape, static_cast<int32_t>(n), qs.data(), ql.data(), cl.data(), co.data(), bt.data(), off.data(),
            batch.q.data(), total, store.keys.data(), store.values.data(), out.data());
    if (st != PB_OK) raise(st);
    return out;
}

/// kvsim::paged_multi_token_attention on the B200 path (attention.hpp:71-72).
template <class Batch, class Store>
std::vector<float> paged_multi_token_attention(const Batch& batch, const Store& store, pb_dtype dtype = PB_F32) {
    return attention(batch, store, false, dtype);
}

/// kvsim::single_token_attention on the B200 path (attention.hpp:76-77).
template <class Batch, class Store>
std::vector<float> single_token_attention(const Batch& batch, const Store& store, pb_dtype dtype = PB_F32) {
    return attention(batch, store, true, dtype);
}

} // namespace pensieve_b200
