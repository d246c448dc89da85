// TEST INFRASTRUCTURE ONLY — the drop-in check from the reference's side.
//
// A kvsim program (reference headers + reference sources, unmodified) calls the B200 path
// through include/pensieve_b200_kvsim.hpp exactly where it would call
// kvsim::paged_multi_token_attention / single_token_attention, and compares:
//   --no-gpu : error behaviour only (validation happens on the host before any launch):
//              NaN query -> kvsim::NumericError, short table / bad context ->
//              kvsim::DimensionMismatch, out-of-range slot -> kvsim::Error, q_len > 1 on the
//              single-token path -> kvsim::DimensionMismatch;
//   default  : also values on acceptance-style instances (proj/tests/acceptance.cpp:100-166
//              shapes): fp32 mode within 1e-5 of kvsim, bf16 mode within 2e-2 + 1e-2|ref|.
// Built by oracle/Makefile into oracle/_ref/kvsim_dropin_test.
#include "kvsim/attention.hpp"
#include "kvsim/errors.hpp"
#include "kvsim/workload.hpp"
#include "pensieve_b200_kvsim.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <numeric>
#include <vector>

using namespace kvsim;

namespace {

int g_fail = 0;
void report(bool ok, const char* what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++g_fail;
}

float unit(SplitMix64& r) { return static_cast<float>(2.0 * r.u01() - 1.0); }

struct Inst {
    PagedKvStore store;
    RaggedQueryBatch batch;
};

Inst make(SplitMix64& rng, int n_head, int n_kv, int hs, int chunk, int n_subs, int max_ctx, bool decode) {
    Inst in;
    std::vector<TokenCount> ctx, ql;
    int slots = 0;
    for (int s = 0; s < n_subs; ++s) {
        TokenCount c = 1 + static_cast<TokenCount>(rng.next() % max_ctx);
        TokenCount q = decode ? 1 : 1 + static_cast<TokenCount>(rng.next() % std::min<TokenCount>(c, 64));
        ctx.push_back(c);
        ql.push_back(q);
        slots += static_cast<int>((c + chunk - 1) / chunk);
    }
    in.store = PagedKvStore(chunk, n_kv, hs, slots + 2);
    for (auto& x : in.store.keys) x = unit(rng);
    for (auto& x : in.store.values) x = unit(rng);
    std::vector<SlotId> pool(static_cast<size_t>(in.store.n_slots));
    std::iota(pool.begin(), pool.end(), 0);
    for (size_t i = pool.size(); i > 1; --i) std::swap(pool[i - 1], pool[rng.next() % i]);
    in.batch.n_head = n_head;
    in.batch.head_size = hs;
    in.batch.scale = std::sqrt(static_cast<double>(hs));
    size_t next = 0;
    TokenCount start = 0;
    for (int s = 0; s < n_subs; ++s) {
        SubRequest sub;
        sub.req_id = s;
        sub.query_start = start;
        sub.query_len = ql[static_cast<size_t>(s)];
        sub.context_len = ctx[static_cast<size_t>(s)];
        sub.causal_offset = sub.context_len - sub.query_len;
        for (TokenCount t = 0; t < (sub.context_len + chunk - 1) / chunk; ++t) sub.block_table.push_back(pool[next++]);
        start += sub.query_len;
        in.batch.sub_requests.push_back(sub);
    }
    in.batch.q.resize(static_cast<size_t>(start) * n_head * hs);
    for (auto& x : in.batch.q) x = unit(rng);
    return in;
}

template <class Ex, class F> bool throws_as(F&& f) {
    try {
        f();
    } catch (const Ex&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

float bf16_round(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&f, &u, 4);
    return f;
}

} // namespace

int main(int argc, char** argv) {
    const bool gpu = !(argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0);
    SplitMix64 rng{20261017};

    // ---- error behaviour (host-side validation, no GPU needed) ----
    {
        Inst in = make(rng, 4, 2, 8, 16, 2, 64, false);
        Inst nan = in;
        nan.batch.q[3] = std::numeric_limits<float>::quiet_NaN();
        report(throws_as<NumericError>([&] { pensieve_b200::paged_multi_token_attention(nan.batch, nan.store); }) &&
                   throws_as<NumericError>([&] { paged_multi_token_attention(nan.batch, nan.store); }),
               "NaN query -> kvsim::NumericError (both paths)");
        Inst shortt = in;
        shortt.batch.sub_requests[0].block_table.clear();
        report(throws_as<DimensionMismatch>([&] { pensieve_b200::paged_multi_token_attention(shortt.batch, shortt.store); }),
               "short block table -> kvsim::DimensionMismatch");
        Inst badctx = in;
        badctx.batch.sub_requests[0].context_len += 1;
        report(throws_as<DimensionMismatch>([&] { pensieve_b200::paged_multi_token_attention(badctx.batch, badctx.store); }),
               "context_len != causal_offset + query_len -> kvsim::DimensionMismatch");
        Inst oob = in;
        oob.batch.sub_requests[0].block_table[0] = oob.store.n_slots + 5;
        report(throws_as<Error>([&] { pensieve_b200::paged_multi_token_attention(oob.batch, oob.store); }) &&
                   !throws_as<DimensionMismatch>([&] { pensieve_b200::paged_multi_token_attention(oob.batch, oob.store); }),
               "out-of-range slot -> kvsim::Error");
        Inst knan = in;
        const auto& s0 = knan.batch.sub_requests[0];
        knan.store.key_row(s0.block_table[0], 0)[0] = std::numeric_limits<float>::infinity();
        report(throws_as<NumericError>([&] { pensieve_b200::paged_multi_token_attention(knan.batch, knan.store); }),
               "non-finite k_row[0] -> kvsim::NumericError");
        bool any_long = false;
        for (const auto& s : in.batch.sub_requests) any_long |= s.query_len > 1;
        if (any_long)
            report(throws_as<DimensionMismatch>([&] { pensieve_b200::single_token_attention(in.batch, in.store); }),
                   "single-token path rejects query_len > 1 -> kvsim::DimensionMismatch");
    }
    if (!gpu) {
        std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ok", g_fail);
        return g_fail ? 1 : 0;
    }

    // ---- values: fp32 validation mode vs kvsim, bf16 mode vs kvsim on bf16-rounded inputs ----
    const int pairs[][2] = {{1, 1}, {3, 3}, {8, 8}, {2, 1}, {4, 2}, {8, 4}, {4, 1}, {8, 2}};
    double worst32 = 0, worst16 = 0;
    bool ok32 = true, ok16 = true, ok_single = true;
    for (int trial = 0; trial < 24; ++trial) {
        const auto& pr = pairs[rng.next() % 8];
        const bool dec = trial % 3 == 2;
        const int hs = trial % 2 ? 128 : 64;
        Inst in = make(rng, pr[0], pr[1], hs, 16, 1 + static_cast<int>(rng.next() % 4), 1500, dec);
        const auto ref = paged_multi_token_attention(in.batch, in.store);
        const auto got = pensieve_b200::paged_multi_token_attention(in.batch, in.store, PB_F32);
        for (size_t i = 0; i < ref.size(); ++i) {
            const double e = std::fabs(static_cast<double>(ref[i]) - got[i]);
            worst32 = std::max(worst32, e);
            ok32 &= e <= 1e-5;
        }
        if (dec) {
            const auto single = pensieve_b200::single_token_attention(in.batch, in.store, PB_F32);
            for (size_t i = 0; i < ref.size(); ++i) ok_single &= std::fabs(static_cast<double>(ref[i]) - single[i]) <= 1e-5;
        }
        Inst r16 = in;
        for (auto& x : r16.batch.q) x = bf16_round(x);
        for (auto& x : r16.store.keys) x = bf16_round(x);
        for (auto& x : r16.store.values) x = bf16_round(x);
        const auto ref16 = paged_multi_token_attention(r16.batch, r16.store);
        const auto got16 = pensieve_b200::paged_multi_token_attention(r16.batch, r16.store, PB_BF16);
        for (size_t i = 0; i < ref16.size(); ++i) {
            const double e = std::fabs(static_cast<double>(ref16[i]) - got16[i]);
            worst16 = std::max(worst16, e);
            ok16 &= e <= 2e-2 + 1e-2 * std::fabs(static_cast<double>(ref16[i]));
        }
    }
    char buf[160];
    std::snprintf(buf, sizeof buf, "fp32 mode == kvsim within 1e-5 (max %.3g)", worst32);
    report(ok32, buf);
    report(ok_single, "single_token_attention == kvsim within 1e-5");
    std::snprintf(buf, sizeof buf, "bf16 mode == kvsim(bf16 inputs) within 2e-2+1e-2|ref| (max %.3g)", worst16);
    report(ok16, buf);
    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ok", g_fail);
    return g_fail ? 1 : 0;
}
