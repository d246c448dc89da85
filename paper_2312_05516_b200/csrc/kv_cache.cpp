// Host bookkeeping of the two-tier KV page pool (see kv_cache.hpp).  Each method restates the
// observable behaviour of the corresponding reference method (file:line in
// /root/reference/proj/src/paged_kv_cache.cpp), validated before mutating so that a failure
// leaves the cache untouched, exactly like the reference.
#include "kv_cache.hpp"

#include "pb_common.hpp"

#include <algorithm>
#include <cstdio>
#include <memory>

namespace pb {

// ------------------------------------------------------------------ SlotTier
SlotTier::SlotTier(int32_t capacity) : owner_(static_cast<size_t>(std::max(0, capacity)), -1) {
    free_.reserve(owner_.size());
    for (int32_t s = capacity - 1; s >= 0; --s) free_.push_back(s); // lowest id on top (:12-26)
}

int32_t SlotTier::take(int64_t chunk) {
    int32_t s;
    if (!lazy_.empty()) { // lingering slots first, most recent first (:28-37)
        s = lazy_.back();
        lazy_.pop_back();
    } else {
        s = free_.back();
        free_.pop_back();
    }
    if (s >= 0) owner_[static_cast<size_t>(s)] = chunk;
    ++used_;
    return s;
}

void SlotTier::give_back(int32_t slot) {
    if (slot >= 0 && slot < capacity()) owner_[static_cast<size_t>(slot)] = -1;
    --used_;
    free_.push_back(slot);
}

void SlotTier::give_back_lazy(int32_t slot) {
    if (slot >= 0 && slot < capacity()) owner_[static_cast<size_t>(slot)] = -1;
    --used_;
    lazy_.push_back(slot);
}

std::string SlotTier::check(const char* name) const {
    const int64_t total = static_cast<int64_t>(free_.size()) + static_cast<int64_t>(lazy_.size()) + used_;
    if (total != capacity())
        return std::string(name) + " tier slot conservation violated";
    std::vector<uint8_t> seen(owner_.size(), 0);
    int32_t owned = 0;
    for (size_t s = 0; s < owner_.size(); ++s)
        if (owner_[s] >= 0) {
            seen[s] = 1;
            ++owned;
        }
    if (owned != used_) return std::string(name) + " allocation count out of sync";
    for (const auto* stack : {&free_, &lazy_})
        for (int32_t s : *stack) {
            if (s < 0 || s >= capacity()) return std::string(name) + " slot id out of range";
            if (seen[static_cast<size_t>(s)]) return std::string(name) + " duplicate slot";
            seen[static_cast<size_t>(s)] = 1;
        }
    return "";
}

// ------------------------------------------------------------------ PagedKvCache
PagedKvCache::PagedKvCache(int32_t page_tokens, int32_t device_slots, int32_t host_slots)
    : page_(page_tokens), dev_(device_slots), host_(host_slots) {
    if (page_tokens < 1) fail(PB_ERR_CONFIG, "chunk_size must be >= 1");
    if (device_slots < 0 || host_slots < 0) fail(PB_ERR_CONFIG, "tier capacities must be >= 0");
}

ChunkRec& PagedKvCache::rec(int64_t id) {
    if (id < 0 || id >= static_cast<int64_t>(chunks_.size()) || !chunks_[static_cast<size_t>(id)].live)
        fail(PB_ERR_INVALID_CHUNK_STATE, "unknown chunk id " + std::to_string(id));
    return chunks_[static_cast<size_t>(id)];
}

const ChunkRec& PagedKvCache::chunk(int64_t id) const { return const_cast<PagedKvCache*>(this)->rec(id); }

const PagedKvCache::Conv& PagedKvCache::conv_or_throw(int64_t conv) const {
    auto it = convs_.find(conv);
    if (it == convs_.end()) fail(PB_ERR_UNKNOWN_CONVERSATION, "conversation " + std::to_string(conv));
    return it->second;
}

// allocate: fill the trailing partial chunk, then open new device chunks (:53-96).  The
// conversation entry exists from the first call even if the allocation is then refused.
std::vector<int64_t> PagedKvCache::allocate(int64_t conv, int64_t n_tokens, double now) {
    std::vector<int64_t> created;
    if (n_tokens <= 0) return created;
    Conv& c = convs_[conv];
    int64_t tail = 0;
    if (!c.chunks.empty()) tail = std::min<int64_t>(page_ - rec(c.chunks.back()).n_tokens, n_tokens);
    const int64_t fresh = n_tokens - tail;
    const int64_t need = (fresh + page_ - 1) / page_;
    if (need > dev_.available())
        fail(PB_ERR_INSUFFICIENT_DEVICE_MEMORY, "allocate needs " + std::to_string(need) + " device slots, " +
                                                    std::to_string(dev_.available()) + " available");
    int64_t left = n_tokens;
    if (tail > 0) {
        ChunkRec& last = rec(c.chunks.back());
        last.n_tokens += tail;
        last.last_active = now;
        c.total += tail;
        left -= tail;
    }
    while (left > 0) {
        const int64_t id = static_cast<int64_t>(chunks_.size());
        ChunkRec r;
        r.conv = conv;
        r.start = c.total;
        r.n_tokens = std::min<int64_t>(page_, left);
        r.loc = Loc::Device;
        r.slot = dev_.take(id);
        r.last_active = now;
        r.live = true;
        chunks_.push_back(r);
        ++live_chunks_;
        c.chunks.push_back(id);
        c.total += r.n_tokens;
        left -= r.n_tokens;
        created.push_back(id);
    }
    return created;
}

// layout: Dropped / Host / Device runs in offset order, adjacent kinds merged (:98-127)
std::vector<Segment> PagedKvCache::layout(int64_t conv, int64_t* total_tokens) const {
    const Conv& c = conv_or_throw(conv);
    if (total_tokens) *total_tokens = c.total;
    std::vector<Segment> out;
    for (int64_t id : c.chunks) {
        const ChunkRec& r = chunk(id);
        if (!out.empty() && out.back().kind == r.loc) {
            out.back().chunks.push_back(id);
            out.back().end = r.end();
        } else {
            out.push_back(Segment{r.loc, r.start, r.end(), {id}});
        }
    }
    return out;
}

// apply_evictions (:129-172): validate all, then move in order.
std::vector<SlotMove> PagedKvCache::apply_evictions(const std::vector<int64_t>& victims, bool to_host) {
    int64_t to_host_count = 0;
    for (int64_t id : victims) {
        const ChunkRec& r = chunk(id);
        if (r.loc == Loc::Device) {
            if (to_host) ++to_host_count;
        } else if (r.loc == Loc::Host) {
            if (to_host) fail(PB_ERR_INVALID_CHUNK_STATE, "chunk " + std::to_string(id) + " is already on the host");
        } else {
            fail(PB_ERR_INVALID_CHUNK_STATE, "chunk " + std::to_string(id) + " is already dropped");
        }
    }
    if (to_host_count > host_.n_free())
        fail(PB_ERR_INSUFFICIENT_HOST_MEMORY, "swap-out needs " + std::to_string(to_host_count) + " host slots, " +
                                                  std::to_string(host_.n_free()) + " free");
    std::vector<SlotMove> moves;
    moves.reserve(victims.size());
    for (int64_t id : victims) {
        ChunkRec& r = rec(id);
        if (r.loc == Loc::Device) {
            const int32_t from = r.slot;
            if (to_host) {
                dev_.give_back_lazy(from); // data lingers until the slot is reused
                r.slot = host_.take(id);
                r.loc = Loc::Host;
            } else {
                dev_.give_back(from);
                r.slot = -1;
                r.loc = Loc::Dropped;
            }
            moves.push_back({id, from, r.slot});
        } else { // host -> dropped
            const int32_t from = r.slot;
            host_.give_back(from);
            r.slot = -1;
            r.loc = Loc::Dropped;
            moves.push_back({id, from, -1});
        }
    }
    return moves;
}

// restore (:174-197): host -> device, host slot freed immediately
std::vector<SlotMove> PagedKvCache::restore(const std::vector<int64_t>& ids) {
    for (int64_t id : ids)
        if (chunk(id).loc != Loc::Host)
            fail(PB_ERR_INVALID_CHUNK_STATE, "restore: chunk " + std::to_string(id) + " is not host-resident");
    if (static_cast<int64_t>(ids.size()) > dev_.available())
        fail(PB_ERR_INSUFFICIENT_DEVICE_MEMORY, "restore needs " + std::to_string(ids.size()) + " device slots, " +
                                                    std::to_string(dev_.available()) + " available");
    std::vector<SlotMove> moves;
    moves.reserve(ids.size());
    for (int64_t id : ids) {
        ChunkRec& r = rec(id);
        const int32_t dslot = dev_.take(id);
        const int32_t hslot = r.slot;
        host_.give_back(hslot);
        r.loc = Loc::Device;
        r.slot = dslot;
        moves.push_back({id, hslot, dslot});
    }
    return moves;
}

// rematerialize (:199-220): dropped -> fresh device slot for recomputation
std::vector<SlotMove> PagedKvCache::rematerialize(const std::vector<int64_t>& ids) {
    for (int64_t id : ids)
        if (chunk(id).loc != Loc::Dropped)
            fail(PB_ERR_INVALID_CHUNK_STATE, "rematerialize: chunk " + std::to_string(id) + " is not dropped");
    if (static_cast<int64_t>(ids.size()) > dev_.available())
        fail(PB_ERR_INSUFFICIENT_DEVICE_MEMORY, "rematerialize needs " + std::to_string(ids.size()) +
                                                    " device slots, " + std::to_string(dev_.available()) +
                                                    " available");
    std::vector<SlotMove> moves;
    moves.reserve(ids.size());
    for (int64_t id : ids) {
        ChunkRec& r = rec(id);
        r.slot = dev_.take(id);
        r.loc = Loc::Device;
        moves.push_back({id, -1, r.slot});
    }
    return moves;
}

// release_conversation (:224-246): every chunk freed immediately (not lazily)
void PagedKvCache::release_conversation(int64_t conv) {
    auto it = convs_.find(conv);
    if (it == convs_.end()) fail(PB_ERR_UNKNOWN_CONVERSATION, "conversation " + std::to_string(conv));
    for (int64_t id : it->second.chunks) {
        ChunkRec& r = rec(id);
        if (r.loc == Loc::Device) dev_.give_back(r.slot);
        else if (r.loc == Loc::Host) host_.give_back(r.slot);
        r.live = false;
        --live_chunks_;
    }
    it->second.chunks.clear();
    it->second.total = 0;
}

void PagedKvCache::touch(int64_t conv, double now) {
    for (int64_t id : conv_or_throw(conv).chunks) rec(id).last_active = now;
}

int64_t PagedKvCache::total_tokens(int64_t conv) const {
    auto it = convs_.find(conv);
    return it == convs_.end() ? 0 : it->second.total;
}

const std::vector<int64_t>& PagedKvCache::conversation_chunks(int64_t conv) const {
    return conv_or_throw(conv).chunks;
}

std::vector<int64_t> PagedKvCache::collect(Loc kind, const std::vector<int64_t>& exclude) const {
    std::vector<int64_t> out;
    for (const auto& [conv, c] : convs_) {
        if (std::find(exclude.begin(), exclude.end(), conv) != exclude.end()) continue;
        for (int64_t id : c.chunks)
            if (chunk(id).loc == kind) out.push_back(id);
    }
    return out;
}

// block_table (:284-304): ceil(ctx/page) device slots, all covered chunks device-resident
std::vector<int32_t> PagedKvCache::block_table(int64_t conv, int64_t context_tokens) const {
    const Conv& c = conv_or_throw(conv);
    if (context_tokens > c.total)
        fail(PB_ERR_ERROR, "block_table: context " + std::to_string(context_tokens) +
                               " exceeds conversation tokens " + std::to_string(c.total));
    std::vector<int32_t> out;
    out.reserve(static_cast<size_t>((context_tokens + page_ - 1) / page_));
    int64_t covered = 0;
    for (int64_t id : c.chunks) {
        if (covered >= context_tokens) break;
        const ChunkRec& r = chunk(id);
        if (r.loc != Loc::Device)
            fail(PB_ERR_ERROR, "block_table: chunk " + std::to_string(id) + " is not device-resident");
        out.push_back(r.slot);
        covered = r.end();
    }
    return out;
}

int32_t PagedKvCache::append_chunks_needed(int64_t conv, int64_t add) const {
    if (add <= 0) return 0;
    const int64_t t = total_tokens(conv);
    return static_cast<int32_t>((t + add + page_ - 1) / page_ - (t + page_ - 1) / page_);
}

std::string PagedKvCache::dump() const {
    std::string s;
    char buf[160];
    for (const auto& [conv, c] : convs_)
        for (int64_t id : c.chunks) {
            const ChunkRec& r = chunk(id);
            char loc[32];
            if (r.loc == Loc::Device) std::snprintf(loc, sizeof loc, "device:%d", r.slot);
            else if (r.loc == Loc::Host) std::snprintf(loc, sizeof loc, "host:%d", r.slot);
            else std::snprintf(loc, sizeof loc, "dropped");
            std::snprintf(buf, sizeof buf, "%lld %lld %lld %s %.6f\n", static_cast<long long>(id),
                          static_cast<long long>(r.conv), static_cast<long long>(r.start), loc, r.last_active);
            s += buf;
        }
    return s;
}

// verify (:341-396): slot conservation, single-tier residency, contiguous offsets
void PagedKvCache::verify() const {
    for (const auto& [tier, name] : {std::pair<const SlotTier*, const char*>{&dev_, "device"}, {&host_, "host"}}) {
        const std::string e = tier->check(name);
        if (!e.empty()) fail(PB_ERR_ERROR, e);
    }
    int64_t n = 0;
    for (const auto& [conv, c] : convs_) {
        int64_t off = 0;
        for (size_t i = 0; i < c.chunks.size(); ++i) {
            const int64_t id = c.chunks[i];
            const ChunkRec& r = chunk(id);
            ++n;
            if (r.conv != conv) fail(PB_ERR_ERROR, "chunk filed under the wrong conversation");
            if (r.start != off) fail(PB_ERR_ERROR, "non-contiguous chunk offsets");
            if (r.n_tokens < 1 || r.n_tokens > page_) fail(PB_ERR_ERROR, "chunk token count out of range");
            if (i + 1 < c.chunks.size() && r.n_tokens != page_)
                fail(PB_ERR_ERROR, "partial chunk before the end of a conversation");
            off = r.end();
            const bool on_dev = r.loc == Loc::Device && r.slot >= 0 && r.slot < dev_.capacity() && dev_.owner(r.slot) == id;
            const bool on_host = r.loc == Loc::Host && r.slot >= 0 && r.slot < host_.capacity() && host_.owner(r.slot) == id;
            if (r.loc == Loc::Device && !on_dev) fail(PB_ERR_ERROR, "device location out of sync with allocation map");
            if (r.loc == Loc::Host && !on_host) fail(PB_ERR_ERROR, "host location out of sync with allocation map");
        }
        if (off != c.total) fail(PB_ERR_ERROR, "conversation total out of sync");
    }
    if (n != live_chunks_) fail(PB_ERR_ERROR, "orphaned chunk records");
}

} // namespace pb

// ====================================================================== C-ABI
using namespace pb;

struct pb_kv_cache {
    PagedKvCache cache;
};

PagedKvCache& pb_cache_impl(pb_kv_cache* c) { return c->cache; }

namespace {

template <class V> void copy_out(const V& v, typename V::value_type* out, int64_t cap, int64_t* n) {
    if (n) *n = static_cast<int64_t>(v.size());
    if (!out) return;
    for (size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = v[i];
}

void moves_out(const std::vector<SlotMove>& m, pb_slot_move* out) {
    if (!out) return;
    for (size_t i = 0; i < m.size(); ++i) out[i] = {m[i].chunk, m[i].src_slot, m[i].dst_slot};
}

void fill_rec(int64_t id, const ChunkRec& r, pb_chunk_record* o) {
    o->chunk_id = id;
    o->conv_id = r.conv;
    o->start_offset = r.start;
    o->n_tokens = r.n_tokens;
    o->location = static_cast<int32_t>(r.loc);
    o->slot = r.slot;
    o->last_active = r.last_active;
}

} // namespace

extern "C" {

pb_status pb_cache_create(int32_t page_tokens, int32_t device_slots, int32_t host_slots, pb_kv_cache** out) {
    return guarded([&] {
        if (!out) fail(PB_ERR_ERROR, "null out");
        *out = nullptr;
        *out = new pb_kv_cache{PagedKvCache(page_tokens, device_slots, host_slots)};
    });
}

void pb_cache_destroy(pb_kv_cache* c) { delete c; }

pb_status pb_cache_allocate(pb_kv_cache* c, int64_t conv, int64_t n_tokens, double now, int64_t* created,
                            int64_t cap, int64_t* n_created) {
    return guarded([&] { copy_out(c->cache.allocate(conv, n_tokens, now), created, cap, n_created); });
}

pb_status pb_cache_apply_evictions(pb_kv_cache* c, const int64_t* ids, int64_t n, int32_t to_host,
                                   pb_slot_move* moves) {
    return guarded([&] {
        moves_out(c->cache.apply_evictions(std::vector<int64_t>(ids, ids + n), to_host != 0), moves);
    });
}

pb_status pb_cache_restore(pb_kv_cache* c, const int64_t* ids, int64_t n, pb_slot_move* moves) {
    return guarded([&] { moves_out(c->cache.restore(std::vector<int64_t>(ids, ids + n)), moves); });
}

pb_status pb_cache_rematerialize(pb_kv_cache* c, const int64_t* ids, int64_t n, pb_slot_move* moves) {
    return guarded([&] { moves_out(c->cache.rematerialize(std::vector<int64_t>(ids, ids + n)), moves); });
}

pb_status pb_cache_release_conversation(pb_kv_cache* c, int64_t conv) {
    return guarded([&] { c->cache.release_conversation(conv); });
}

pb_status pb_cache_touch(pb_kv_cache* c, int64_t conv, double now) {
    return guarded([&] { c->cache.touch(conv, now); });
}

pb_status pb_cache_block_table(const pb_kv_cache* c, int64_t conv, int64_t context_tokens, int32_t* out,
                               int64_t cap, int64_t* n) {
    return guarded([&] { copy_out(c->cache.block_table(conv, context_tokens), out, cap, n); });
}

pb_status pb_cache_layout(const pb_kv_cache* c, int64_t conv, pb_layout_segment* segs, int64_t cap, int64_t* n,
                          int64_t* total_tokens) {
    return guarded([&] {
        auto L = c->cache.layout(conv, total_tokens);
        if (n) *n = static_cast<int64_t>(L.size());
        for (size_t i = 0; segs && i < L.size() && static_cast<int64_t>(i) < cap; ++i)
            segs[i] = {static_cast<int32_t>(L[i].kind), static_cast<int32_t>(L[i].chunks.size()), L[i].begin,
                       L[i].end, L[i].chunks.front()};
    });
}

pb_status pb_cache_conversation_chunks(const pb_kv_cache* c, int64_t conv, pb_chunk_record* out, int64_t cap,
                                       int64_t* n) {
    return guarded([&] {
        const auto& ids = c->cache.conversation_chunks(conv);
        if (n) *n = static_cast<int64_t>(ids.size());
        for (size_t i = 0; out && i < ids.size() && static_cast<int64_t>(i) < cap; ++i)
            fill_rec(ids[i], c->cache.chunk(ids[i]), &out[i]);
    });
}

pb_status pb_cache_chunk(const pb_kv_cache* c, int64_t id, pb_chunk_record* out) {
    return guarded([&] { fill_rec(id, c->cache.chunk(id), out); });
}

pb_status pb_cache_collect_chunks(const pb_kv_cache* c, int32_t location, const int64_t* exclude_convs,
                                  int64_t n_exclude, int64_t* ids, int64_t cap, int64_t* n) {
    return guarded([&] {
        std::vector<int64_t> ex(exclude_convs, exclude_convs + (exclude_convs ? n_exclude : 0));
        copy_out(c->cache.collect(static_cast<Loc>(location), ex), ids, cap, n);
    });
}

void pb_cache_counts(const pb_kv_cache* c, int64_t* o) {
    const auto& d = c->cache.device();
    const auto& h = c->cache.host();
    o[0] = d.capacity();
    o[1] = d.n_free();
    o[2] = d.n_lazy();
    o[3] = d.n_used();
    o[4] = h.capacity();
    o[5] = h.n_free();
    o[6] = h.n_used();
    o[7] = c->cache.page_tokens();
}

int32_t pb_cache_has_conversation(const pb_kv_cache* c, int64_t conv) {
    return c->cache.has_conversation(conv) ? 1 : 0;
}

int64_t pb_cache_total_tokens(const pb_kv_cache* c, int64_t conv) { return c->cache.total_tokens(conv); }

int32_t pb_cache_append_chunks_needed(const pb_kv_cache* c, int64_t conv, int64_t add) {
    return c->cache.append_chunks_needed(conv, add);
}

pb_status pb_cache_verify(const pb_kv_cache* c) {
    return guarded([&] { c->cache.verify(); });
}

int64_t pb_cache_dump(const pb_kv_cache* c, char* buf, int64_t cap) {
    const std::string s = c->cache.dump();
    if (buf && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::copy(s.data(), s.data() + n, buf);
        buf[n] = '\0';
    }
    return static_cast<int64_t>(s.size());
}

} // extern "C"
