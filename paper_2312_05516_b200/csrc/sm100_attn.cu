// placeholder: replaced by the tcgen05 tile kernel
#include "sm100_attn.hpp"
#include "pb_common.hpp"
namespace pb {
bool sm100_supports(int, int, int) { return false; }
int sm100_tile_tokens(int group) { return 128 / group; }
void launch_attn_sm100(const AttnParams&, const pb_attn_shape&, Sm100Cache&, int64_t, cudaStream_t) {
    fail(PB_ERR_UNSUPPORTED, "sm100 path not built");
}
void sm100_cache_release(Sm100Cache&) {}
}
