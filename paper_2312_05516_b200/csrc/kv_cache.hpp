// Two-tier (HBM / pinned host) KV page-slot bookkeeping with the exact slot semantics of the
// reference PagedKvCache (/root/reference/proj/include/kvsim/paged_kv_cache.hpp:52-153,
// src/paged_kv_cache.cpp), so block tables and swap slot lists are bit-identical.  What the
// B200 build adds is slot-pair reporting: every tier move also reports (chunk, source slot,
// destination slot), which the reference drops (restore frees the host slot, :190;
// apply_evictions forgets the device slot, :155-161) but a copy engine needs.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

namespace pb {

enum class Loc : int8_t { Device = 0, Host = 1, Dropped = 2 };

struct ChunkRec {
    int64_t conv = -1;
    int64_t start = 0;    // first token position covered
    int64_t n_tokens = 0; // tokens stored (<= page size)
    Loc loc = Loc::Dropped;
    int32_t slot = -1;
    double last_active = 0.0;
    bool live = false;
    int64_t end() const { return start + n_tokens; }
};

struct SlotMove {
    int64_t chunk;
    int32_t src_slot; // tier the chunk left (-1 when dropped data is rematerialised)
    int32_t dst_slot; // tier the chunk entered (-1 when dropped)
};

struct Segment {
    Loc kind;        // Dropped = recompute, Host = swap in, Device = resident
    int64_t begin, end;
    std::vector<int64_t> chunks;
};

// One tier's slots: a LIFO free stack that hands out the lowest ids first, plus a LIFO
// "lazy" stack of device slots vacated by swap-out whose data still lingers; lazy slots are
// reused before free ones (reference TierState::acquire, src/paged_kv_cache.cpp:28-37).
class SlotTier {
public:
    explicit SlotTier(int32_t capacity = 0);
    int32_t capacity() const { return static_cast<int32_t>(owner_.size()); }
    int32_t n_free() const { return static_cast<int32_t>(free_.size()); }
    int32_t n_lazy() const { return static_cast<int32_t>(lazy_.size()); }
    int32_t n_used() const { return used_; }
    int32_t available() const { return n_free() + n_lazy(); }
    int32_t take(int64_t chunk);         // lazy first, then free
    void give_back(int32_t slot);        // -> free stack
    void give_back_lazy(int32_t slot);   // -> lazy stack
    int64_t owner(int32_t slot) const { return owner_[static_cast<size_t>(slot)]; }
    std::string check(const char* name) const;

private:
    std::vector<int32_t> free_, lazy_;
    std::vector<int64_t> owner_; // chunk id per slot, -1 if not allocated
    int32_t used_ = 0;
};

class PagedKvCache {
public:
    PagedKvCache(int32_t page_tokens, int32_t device_slots, int32_t host_slots);

    int32_t page_tokens() const { return page_; }
    const SlotTier& device() const { return dev_; }
    const SlotTier& host() const { return host_; }

    std::vector<int64_t> allocate(int64_t conv, int64_t n_tokens, double now);
    std::vector<Segment> layout(int64_t conv, int64_t* total_tokens) const;
    // to_host: device -> host (device slot becomes lazy); else -> dropped (slots freed)
    std::vector<SlotMove> apply_evictions(const std::vector<int64_t>& victims, bool to_host);
    std::vector<SlotMove> restore(const std::vector<int64_t>& chunks);       // host -> device
    std::vector<SlotMove> rematerialize(const std::vector<int64_t>& chunks); // dropped -> device
    void release_conversation(int64_t conv);
    void touch(int64_t conv, double now);
    bool has_conversation(int64_t conv) const { return convs_.count(conv) != 0; }
    int64_t total_tokens(int64_t conv) const;
    const ChunkRec& chunk(int64_t id) const;
    const std::vector<int64_t>& conversation_chunks(int64_t conv) const;
    std::vector<int64_t> collect(Loc kind, const std::vector<int64_t>& exclude_convs) const;
    std::vector<int32_t> block_table(int64_t conv, int64_t context_tokens) const;
    int32_t append_chunks_needed(int64_t conv, int64_t add) const;
    std::string dump() const;
    void verify() const; // throws Failure(PB_ERR_ERROR) on any invariant violation

private:
    struct Conv {
        std::vector<int64_t> chunks;
        int64_t total = 0;
    };
    ChunkRec& rec(int64_t id);
    const Conv& conv_or_throw(int64_t conv) const;

    int32_t page_;
    SlotTier dev_, host_;
    std::map<int64_t, Conv> convs_;   // ordered: deterministic scans and dumps
    std::vector<ChunkRec> chunks_;    // indexed by chunk id (ids are handed out densely)
    int64_t live_chunks_ = 0;
};

} // namespace pb

struct pb_kv_cache;
pb::PagedKvCache& pb_cache_impl(pb_kv_cache* c); // C-ABI handle -> C++ object
