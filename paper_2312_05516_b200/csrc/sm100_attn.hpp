// sm_100a tile path of the fused ragged paged attention (see sm100_attn.cu).
#pragma once

#include "attn_internal.hpp"
#include "pensieve_b200.h"

#include <cuda_runtime.h>

#include <cstdint>

namespace pb {

// Host-side cache of the TMA tensor maps of the last launch (re-encoded only when the
// q / page pointers or shapes change).
struct Sm100Cache {
    const void* q = nullptr;
    const void* k = nullptr;
    const void* v = nullptr;
    const void* out = nullptr;
    int64_t total_tokens = -1;
    alignas(64) unsigned char maps[5][128]; // q tiles, k pages, v pages, q decode rows, out tiles
    bool valid = false;
};

bool sm100_supports(int head_size, int chunk, int group);
int sm100_tile_tokens(int group);
void launch_attn_sm100(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache,
                       int64_t total_tokens, cudaStream_t stream);
void sm100_cache_release(Sm100Cache& cache);
// (re)encodes the q / k / v tensor maps when pointers or sizes changed
void sm100_prepare_maps(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens);
bool decode_supports(int head_size, int chunk, int group);
bool decode_tc_supports(int head_size, int chunk, int group);
// stand-alone launch of the fused append's row writes (bf16 rows; paths without the prologue)
void launch_append_spans(const AttnParams& p, cudaStream_t stream);
void launch_attn_decode_tc(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache,
                           int64_t total_tokens, cudaStream_t stream);
void launch_attn_decode(const AttnParams& p, const pb_attn_shape& shape, Sm100Cache& cache, int64_t total_tokens,
                        cudaStream_t stream);

} // namespace pb
