// ModelConfig byte arithmetic and the KV-head shard geometry of the
// multi-GPU control plane.
//
// Semantics: kvsim::ModelConfig::validate / kv_token_bytes / chunk_bytes / preset,
// /root/reference/proj/src/model_config.cpp:13-68.  chunk_bytes is the PER-WORKER size of one
// chunk: the KV heads are split over n_partitions workers, each holding n_kv_head/n_partitions
// heads of every layer (:36-40), which is exactly what one rank's page pools and host tier
// hold under pb_shard_shape, so pb_tier_chunk_bytes of a rank's tier equals it.
#include "pb_common.hpp"

#include <cstring>
#include <string>

using namespace pb;

namespace {

void validate_model(const pb_model_config& m) { // model_config.cpp:13-27, same order
    if (m.n_layer < 0) fail(PB_ERR_CONFIG, "n_layer must be >= 0");
    if (m.n_head <= 0 || m.n_kv_head <= 0 || m.head_size <= 0)
        fail(PB_ERR_CONFIG, "head counts and head_size must be positive");
    if (m.hidden != m.n_head * m.head_size) fail(PB_ERR_CONFIG, "hidden must equal n_head * head_size");
    if (m.n_head % m.n_kv_head != 0) fail(PB_ERR_CONFIG, "n_head must be a multiple of n_kv_head");
    if (m.bytes_per_scalar <= 0) fail(PB_ERR_CONFIG, "bytes_per_scalar must be positive");
    if (m.n_partitions < 1) fail(PB_ERR_CONFIG, "n_partitions must be >= 1");
    if (m.n_kv_head % m.n_partitions != 0) fail(PB_ERR_CONFIG, "n_kv_head must be divisible by n_partitions");
}

uint64_t kv_token_bytes(const pb_model_config& m) { // :29-34, keys and values, every layer
    return 2ull * static_cast<uint64_t>(m.n_layer) * static_cast<uint64_t>(m.n_kv_head) *
           static_cast<uint64_t>(m.head_size) * static_cast<uint64_t>(m.bytes_per_scalar);
}

} // namespace

extern "C" {

pb_status pb_model_validate(const pb_model_config* m) {
    return guarded([&] {
        if (!m) fail(PB_ERR_ERROR, "null model config");
        validate_model(*m);
    });
}

pb_status pb_model_kv_token_bytes(const pb_model_config* m, uint64_t* out) {
    return guarded([&] {
        if (!m || !out) fail(PB_ERR_ERROR, "null argument");
        *out = kv_token_bytes(*m);
    });
}

pb_status pb_model_chunk_bytes(const pb_model_config* m, int32_t chunk_size, uint64_t* out) {
    return guarded([&] { // :36-40
        if (!m || !out) fail(PB_ERR_ERROR, "null argument");
        if (chunk_size < 1) fail(PB_ERR_CONFIG, "chunk_size must be >= 1");
        if (m->n_partitions < 1) fail(PB_ERR_CONFIG, "n_partitions must be >= 1"); // ref: division by zero
        *out = kv_token_bytes(*m) * static_cast<uint64_t>(chunk_size) / static_cast<uint64_t>(m->n_partitions);
    });
}

pb_status pb_model_preset(const char* name, pb_model_config* out) {
    return guarded([&] { // :48-68
        if (!name || !out) fail(PB_ERR_ERROR, "null argument");
        pb_model_config c{};
        c.bytes_per_scalar = 2;
        const std::string n = name;
        if (n == "opt-13b") c = {40, 5120, 40, 40, 128, 2, 1};
        else if (n == "opt-66b") c = {64, 9216, 72, 72, 128, 2, 4};
        else if (n == "llama2-13b") c = {40, 5120, 40, 10, 128, 2, 1};
        else if (n == "llama2-70b") c = {80, 8192, 64, 8, 128, 2, 4};
        else fail(PB_ERR_CONFIG, "unknown model preset: " + n);
        validate_model(c);
        *out = c;
    });
}

pb_status pb_shard_shape(const pb_attn_shape* full, int32_t rank, int32_t world, pb_attn_shape* out,
                         int32_t* first_head, int32_t* first_kv_head) {
    return guarded([&] {
        if (!full || !out) fail(PB_ERR_ERROR, "null argument");
        if (world < 1 || rank < 0 || rank >= world) fail(PB_ERR_CONFIG, "rank must be in [0, world)");
        if (full->n_kv_head <= 0 || full->n_head <= 0 || full->n_head % full->n_kv_head != 0)
            fail(PB_ERR_DIMENSION_MISMATCH, "n_head must be a positive multiple of n_kv_head");
        // model_config.cpp:25-26: the KV heads must split evenly over the workers
        if (full->n_kv_head % world != 0)
            fail(PB_ERR_DIMENSION_MISMATCH, "n_kv_head must be divisible by the number of partitions");
        pb_attn_shape s = *full;
        s.n_kv_head = full->n_kv_head / world;
        s.n_head = full->n_head / world; // head h reads kv head h / group: a contiguous block
        *out = s;
        if (first_head) *first_head = rank * s.n_head;
        if (first_kv_head) *first_kv_head = rank * s.n_kv_head;
    });
}

} // extern "C"
