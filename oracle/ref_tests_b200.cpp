// TEST INFRASTRUCTURE ONLY.  Runs the reference's OWN attention unit tests
// (/root/reference/proj/tests/test_attention.cpp, compiled unchanged) against the B200 path:
// oracle/Makefile weakens kvsim::paged_multi_token_attention and kvsim::single_token_attention
// in the reference's attention.o (objcopy --weaken-symbol) and links these definitions, which
// forward through the drop-in adapter (include/pensieve_b200_kvsim.hpp) to the C-ABI library in
// fp32 validation mode.  Everything else in those tests (dense oracle, copy-out straw-man,
// qkv_project, fixtures) stays the reference's own code.
#include "kvsim/attention.hpp"
#include "pensieve_b200_kvsim.hpp"

namespace kvsim {

std::vector<float> paged_multi_token_attention(const RaggedQueryBatch& batch, const PagedKvStore& store) {
    return pensieve_b200::paged_multi_token_attention(batch, store, PB_F32);
}

std::vector<float> single_token_attention(const RaggedQueryBatch& batch, const PagedKvStore& store) {
    return pensieve_b200::single_token_attention(batch, store, PB_F32);
}

} // namespace kvsim
