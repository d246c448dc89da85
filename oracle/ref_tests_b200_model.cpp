// TEST INFRASTRUCTURE ONLY.  Runs the reference's OWN ModelConfig unit tests
// (/root/reference/proj/tests/test_model_config.cpp, compiled unchanged) against this repo's
// byte arithmetic: oracle/Makefile weakens ModelConfig::validate,
// kv_token_bytes, chunk_bytes and preset in the reference's model_config.o and links these
// definitions, which call the C-ABI (pb_model_*, csrc/model_config.cpp) and rethrow its status
// as the reference's exceptions (include/pensieve_b200_kvsim.hpp).  load / to_text (file I/O,
// out of scope) stay the reference's, and call the substituted validate.
#include "kvsim/model_config.hpp"
#include "pensieve_b200_kvsim.hpp"

namespace {
pb_model_config to_pb(const kvsim::ModelConfig& m) {
    return pb_model_config{m.n_layer, m.hidden, m.n_head, m.n_kv_head, m.head_size, m.bytes_per_scalar,
                           m.n_partitions};
}
void check(pb_status st) {
    if (st != PB_OK) pensieve_b200::raise(st);
}
} // namespace

namespace kvsim {

void ModelConfig::validate() const {
    const pb_model_config c = to_pb(*this);
    check(pb_model_validate(&c));
}

std::uint64_t ModelConfig::kv_token_bytes() const {
    const pb_model_config c = to_pb(*this);
    uint64_t v = 0;
    check(pb_model_kv_token_bytes(&c, &v));
    return v;
}

std::uint64_t ModelConfig::chunk_bytes(int chunk_size) const {
    const pb_model_config c = to_pb(*this);
    uint64_t v = 0;
    check(pb_model_chunk_bytes(&c, chunk_size, &v));
    return v;
}

ModelConfig ModelConfig::preset(const std::string& name) {
    pb_model_config c{};
    check(pb_model_preset(name.c_str(), &c));
    ModelConfig m;
    m.name = name;
    m.n_layer = c.n_layer;
    m.hidden = c.hidden;
    m.n_head = c.n_head;
    m.n_kv_head = c.n_kv_head;
    m.head_size = c.head_size;
    m.bytes_per_scalar = c.bytes_per_scalar;
    m.n_partitions = c.n_partitions;
    return m;
}

} // namespace kvsim
