// control.cpp — native host control-plane streams (include/mecefo_ctl.h).
//
// Bit-exact restatement of the numpy streams the reference's integer path draws
// from (reference pkg/src/faultsim/cluster.py:98,149,164 and data.py:96,104):
// SeedSequence (NEP 19 hash pool of 4 uint32 words), PCG64 XSL-RR 128/64,
// Generator.random() and Generator.integers() (Lemire's nearly-divisionless
// bounded draw; 32-bit ranges go through numpy's buffered next_uint32).
// Checked draw-for-draw against numpy in tests/test_control_native.py.

#include "mecefo_ctl.h"


namespace {

typedef unsigned __int128 u128;

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;
const u128 kPcgMult = (static_cast<u128>(0x2360ed051fc65da4ull) << 64) | 0x4385df649fccf645ull;

inline uint32_t hashmix(uint32_t v, uint32_t& h) {
    v ^= h;
    h *= kMultA;
    v *= h;
    v ^= v >> 16;
    return v;
}

inline uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = kMixL * x - kMixR * y;
    return r ^ (r >> 16);
}

// SeedSequence(entropy) -> generate_state(4, uint64) as 8 uint32 words.
void seed_sequence_state(const uint64_t* ent, int n, uint32_t out[8]) {
    uint32_t words[128];  // _coerce_to_uint32_array: each int -> LE 32-bit words, 0 -> [0]
    int nw = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t v = ent[i];
        if (v == 0) words[nw++] = 0;
        while (v) {
            words[nw++] = static_cast<uint32_t>(v);
            v >>= 32;
        }
    }
    uint32_t pool[kPool];
    uint32_t h = kInitA;
    for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < nw ? words[i] : 0u, h);
    for (int s = 0; s < kPool; ++s)
        for (int d = 0; d < kPool; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
    for (int s = kPool; s < nw; ++s)
        for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(words[s], h));
    uint32_t hb = kInitB;
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i % kPool];
        v ^= hb;
        hb *= kMultB;
        v *= hb;
        v ^= v >> 16;
        out[i] = v;
    }
}

inline u128 get_state(const mecefo_pcg64_t* s) { return (static_cast<u128>(s->state_hi) << 64) | s->state_lo; }
inline u128 get_inc(const mecefo_pcg64_t* s) { return (static_cast<u128>(s->inc_hi) << 64) | s->inc_lo; }
inline void put_state(mecefo_pcg64_t* s, u128 v) {
    s->state_hi = static_cast<uint64_t>(v >> 64);
    s->state_lo = static_cast<uint64_t>(v);
}

inline uint64_t next64(mecefo_pcg64_t* s) {
    u128 st = get_state(s) * kPcgMult + get_inc(s);
    put_state(s, st);
    uint64_t hi = static_cast<uint64_t>(st >> 64), lo = static_cast<uint64_t>(st);
    unsigned rot = static_cast<unsigned>(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

inline uint32_t next32(mecefo_pcg64_t* s) {
    if (s->has_uint32) {
        s->has_uint32 = 0;
        return s->uinteger;
    }
    uint64_t v = next64(s);
    s->has_uint32 = 1;
    s->uinteger = static_cast<uint32_t>(v >> 32);
    return static_cast<uint32_t>(v);
}

// numpy random/src/distributions/distributions.c: buffered_bounded_lemire_uint32
inline uint32_t lemire32(mecefo_pcg64_t* s, uint32_t rng) {
    const uint32_t excl = rng + 1u;
    uint64_t m = static_cast<uint64_t>(next32(s)) * excl;
    uint32_t left = static_cast<uint32_t>(m);
    if (left < excl) {
        const uint32_t thr = (0xffffffffu - rng) % excl;
        while (left < thr) {
            m = static_cast<uint64_t>(next32(s)) * excl;
            left = static_cast<uint32_t>(m);
        }
    }
    return static_cast<uint32_t>(m >> 32);
}

// bounded_lemire_uint64
inline uint64_t lemire64(mecefo_pcg64_t* s, uint64_t rng) {
    const uint64_t excl = rng + 1u;
    u128 m = static_cast<u128>(next64(s)) * excl;
    uint64_t left = static_cast<uint64_t>(m);
    if (left < excl) {
        const uint64_t thr = (0xffffffffffffffffull - rng) % excl;
        while (left < thr) {
            m = static_cast<u128>(next64(s)) * excl;
            left = static_cast<uint64_t>(m);
        }
    }
    return static_cast<uint64_t>(m >> 64);
}

}  // namespace

extern "C" {

int mecefo_pcg64_seed(mecefo_pcg64_t* s, const uint64_t* entropy, int32_t n) {
    if (!s || !entropy || n < 1 || n > 64) return MECEFO_CTL_CONTRACT;
    uint32_t w[8];
    seed_sequence_state(entropy, n, w);
    // generate_state(4, uint64) viewed little-endian; pcg64_set_seed(seed=v[0:2], inc=v[2:4])
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = static_cast<uint64_t>(w[2 * i]) | (static_cast<uint64_t>(w[2 * i + 1]) << 32);
    const u128 initstate = (static_cast<u128>(v[0]) << 64) | v[1];
    const u128 initseq = (static_cast<u128>(v[2]) << 64) | v[3];
    const u128 inc = (initseq << 1) | 1u;
    s->inc_hi = static_cast<uint64_t>(inc >> 64);
    s->inc_lo = static_cast<uint64_t>(inc);
    put_state(s, 0);
    put_state(s, get_state(s) * kPcgMult + inc);
    put_state(s, get_state(s) + initstate);
    put_state(s, get_state(s) * kPcgMult + inc);
    s->has_uint32 = 0;
    s->uinteger = 0;
    return MECEFO_CTL_OK;
}

int mecefo_pcg64_next_u64(mecefo_pcg64_t* s, uint64_t* out, size_t count) {
    if (!s || (count && !out)) return MECEFO_CTL_CONTRACT;
    for (size_t i = 0; i < count; ++i) out[i] = next64(s);
    return MECEFO_CTL_OK;
}

int mecefo_pcg64_next_u32(mecefo_pcg64_t* s, uint32_t* out, size_t count) {
    if (!s || (count && !out)) return MECEFO_CTL_CONTRACT;
    for (size_t i = 0; i < count; ++i) out[i] = next32(s);
    return MECEFO_CTL_OK;
}

int mecefo_pcg64_random(mecefo_pcg64_t* s, double* out, size_t count) {
    if (!s || (count && !out)) return MECEFO_CTL_CONTRACT;
    for (size_t i = 0; i < count; ++i) out[i] = static_cast<double>(next64(s) >> 11) * (1.0 / 9007199254740992.0);
    return MECEFO_CTL_OK;
}

int mecefo_pcg64_integers(mecefo_pcg64_t* s, int64_t low, int64_t high, int64_t* out, size_t count) {
    if (!s || (count && !out) || high <= low) return MECEFO_CTL_CONTRACT;
    const uint64_t rng = static_cast<uint64_t>(high) - static_cast<uint64_t>(low) - 1u;
    if (rng == 0) {
        for (size_t i = 0; i < count; ++i) out[i] = low;
    } else if (rng <= 0xffffffffull) {
        if (rng == 0xffffffffull) {
            for (size_t i = 0; i < count; ++i) out[i] = low + static_cast<int64_t>(next32(s));
        } else {
            for (size_t i = 0; i < count; ++i) out[i] = low + static_cast<int64_t>(lemire32(s, static_cast<uint32_t>(rng)));
        }
    } else if (rng == 0xffffffffffffffffull) {
        for (size_t i = 0; i < count; ++i) out[i] = static_cast<int64_t>(static_cast<uint64_t>(low) + next64(s));
    } else {
        for (size_t i = 0; i < count; ++i) out[i] = static_cast<int64_t>(static_cast<uint64_t>(low) + lemire64(s, rng));
    }
    return MECEFO_CTL_OK;
}

int mecefo_ring_route(int32_t n, const uint8_t* failed, int32_t* executor) {
    if (n < 1 || !failed || !executor) return MECEFO_CTL_CONTRACT;
    // adopting[t]: t already runs one failed member's work (one adoption each)
    uint8_t stackbuf[256];
    uint8_t* adopting = n <= 256 ? stackbuf : new uint8_t[n];
    for (int32_t j = 0; j < n; ++j) {
        adopting[j] = 0;
        executor[j] = j;
    }
    int rc = MECEFO_CTL_OK;
    for (int32_t s = n - 1; s >= 0 && rc == MECEFO_CTL_OK; --s) {
        if (!failed[s]) continue;
        int32_t hop = 1, t = (s + 1) % n;
        while (hop < n && (failed[t] || adopting[t])) {
            ++hop;
            t = (s + hop) % n;
        }
        if (hop >= n) {
            rc = MECEFO_CTL_UNRECOVERABLE;
        } else {
            adopting[t] = 1;
            executor[s] = t;
        }
    }
    if (adopting != stackbuf) delete[] adopting;
    return rc;
}

}  // extern "C"
