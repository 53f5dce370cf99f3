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

// ---------------------------------------------------------------------------
// The cluster state machine (reference cluster.py:92-271): node health,
// executor map, recovery deadlines, failure injection (per-iteration coin
// flips or scheduled interval crossings on the simulated clock), ring-successor
// NDB reassignment and the partition invariants — and iteration_cost
// (costmodel.py:206-238), whose FLOP total drives the simulated clock that
// scheduled failures key on (harness.py:442-446). Mirrors the Python control
// plane that is replayed bit-exactly against the reference's own logs.
// ---------------------------------------------------------------------------

#include <algorithm>
#include <cmath>
#include <map>
#include <new>
#include <vector>

struct mecefo_cluster {
    int32_t dp = 0, pp = 0, layers = 0;
    std::vector<int32_t> bounds;        // pp + 1 stage boundaries
    int32_t kind = 0;                   // 0 none, 1 per_iteration, 2 scheduled
    double probability = 0.0;
    int32_t recovery_iterations = 1;
    double failure_interval_s = 0.0, recovery_time_s = 0.0;
    bool has_victims = false;
    std::vector<uint8_t> victim;        // dp * pp
    mecefo_pcg64_t rng{};
    std::vector<int8_t> st;             // 0 healthy, 1 failed, 2 doubled
    std::vector<int32_t> ex;            // executing stage within the DP rank
    std::map<int32_t, double> down_until;  // node index i * pp + s -> deadline (iteration or sim time)
    double next_failure_time = 0.0;
};

namespace {

struct EventSink {
    mecefo_cluster_event* out;
    int32_t cap, n;
    int push(const mecefo_cluster_event& e) {
        if (n >= cap) return MECEFO_CTL_CONTRACT;
        out[n++] = e;
        return MECEFO_CTL_OK;
    }
};

mecefo_cluster_event make_event(double t, int32_t it, int32_t kind, int32_t i, int32_t s) {
    mecefo_cluster_event e{};
    e.time = t;
    e.iteration = it;
    e.kind = kind;
    e.node_rank = i;
    e.node_stage = s;
    e.stage = -1;
    e.from_rank = -1;
    e.from_stage = -1;
    return e;
}

// cluster.py:136-168 (only healthy, victim-eligible nodes draw; p == 0 draws nothing)
int inject(mecefo_cluster* c, double sim_time, int32_t iteration, EventSink& ev) {
    if (c->kind == 0) return MECEFO_CTL_OK;
    if (c->kind == 1) {
        if (c->probability == 0.0) return MECEFO_CTL_OK;
        for (int32_t i = 0; i < c->dp; ++i)
            for (int32_t s = 0; s < c->pp; ++s) {
                const int32_t n = i * c->pp + s;
                if (c->st[n] != 0) continue;
                if (c->has_victims && !c->victim[n]) continue;
                double u;
                mecefo_pcg64_random(&c->rng, &u, 1);
                if (u < c->probability) {
                    c->st[n] = 1;
                    c->down_until[n] = (double)iteration + c->recovery_iterations;
                    if (ev.push(make_event(sim_time, iteration, 0, i, s))) return MECEFO_CTL_CONTRACT;
                }
            }
        return MECEFO_CTL_OK;
    }
    while (sim_time >= c->next_failure_time) {
        const double boundary = c->next_failure_time;
        c->next_failure_time += c->failure_interval_s;
        std::vector<int32_t> cands;
        for (int32_t n = 0; n < c->dp * c->pp; ++n)  // row-major == sorted (i, s)
            if (c->st[n] == 0 && (!c->has_victims || c->victim[n])) cands.push_back(n);
        if (cands.empty()) continue;
        int64_t pick;
        mecefo_pcg64_integers(&c->rng, 0, (int64_t)cands.size(), &pick, 1);
        const int32_t n = cands[(size_t)pick];
        c->st[n] = 1;
        c->down_until[n] = boundary + c->recovery_time_s;
        if (ev.push(make_event(boundary, iteration, 0, n / c->pp, n % c->pp))) return MECEFO_CTL_CONTRACT;
    }
    return MECEFO_CTL_OK;
}

// cluster.py:176-187
int recover(mecefo_cluster* c, int32_t i, int32_t s, double sim_time, int32_t iteration, EventSink& ev) {
    const int32_t n = i * c->pp + s;
    if (c->st[n] != 1) return MECEFO_CTL_CONTRACT;
    const int32_t old = c->ex[n];
    c->st[n] = 0;
    c->down_until.erase(n);
    c->ex[n] = s;
    if (old != s && c->st[i * c->pp + old] == 2) {
        int32_t cnt = 0;
        for (int32_t t = 0; t < c->pp; ++t) cnt += c->ex[i * c->pp + t] == old;
        if (cnt == 1) c->st[i * c->pp + old] = 0;
    }
    mecefo_cluster_event e = make_event(sim_time, iteration, 1, i, s);
    e.from_rank = i;
    e.from_stage = old;
    return ev.push(e);
}

// cluster.py:190-239 (descending failed-stage order, ring successor, cascading)
int reassign(mecefo_cluster* c, double sim_time, int32_t iteration, EventSink& ev) {
    std::vector<uint8_t> failed(c->pp);
    std::vector<int32_t> route(c->pp);
    for (int32_t i = 0; i < c->dp; ++i) {
        for (int32_t s = 0; s < c->pp; ++s) failed[s] = c->st[i * c->pp + s] == 1;
        if (mecefo_ring_route(c->pp, failed.data(), route.data()) != MECEFO_CTL_OK) return MECEFO_CTL_UNRECOVERABLE;
        std::vector<uint8_t> adopter(c->pp, 0);
        for (int32_t s = 0; s < c->pp; ++s)
            if (failed[s]) adopter[route[s]] = 1;
        for (int32_t s = 0; s < c->pp; ++s)
            if (!failed[s]) c->ex[i * c->pp + s] = s;
        for (int32_t s = c->pp - 1; s >= 0; --s) {
            if (!failed[s] || c->ex[i * c->pp + s] == route[s]) continue;
            c->ex[i * c->pp + s] = route[s];
            mecefo_cluster_event e = make_event(sim_time, iteration, 2, i, route[s]);
            e.stage = s;
            e.from_rank = c->dp > 1 ? (i + 1) % c->dp : i;
            if (ev.push(e)) return MECEFO_CTL_CONTRACT;
        }
        for (int32_t s = 0; s < c->pp; ++s)
            if (!failed[s]) c->st[i * c->pp + s] = adopter[s] ? 2 : 0;
    }
    return MECEFO_CTL_OK;
}

// cluster.py:253-271
int validate(const mecefo_cluster* c) {
    for (int32_t i = 0; i < c->dp; ++i) {
        std::vector<int32_t> counts(c->pp, 0);
        for (int32_t s = 0; s < c->pp; ++s) {
            const int32_t e = c->ex[i * c->pp + s];
            if (e < 0 || e >= c->pp || c->st[i * c->pp + e] == 1) return 3;
            counts[e]++;
        }
        for (int32_t s = 0; s < c->pp; ++s) {
            const int8_t v = c->st[i * c->pp + s];
            const int32_t want = v == 0 ? 1 : (v == 1 ? 0 : 2);
            if (counts[s] != want) return 3;
        }
    }
    return MECEFO_CTL_OK;
}

// costmodel.py:103-139 totals (linear layers) and :47-64
int64_t svd_flops(int64_t m, int64_t n, int64_t r) {
    const int64_t k = std::min(n, r + 4);
    return 2 * m * n * n + 30 * (2 * n * n * k + 2 * n * k * k);
}

int64_t block_flops(int64_t m, int64_t f, int32_t approx, int64_t r, int64_t tau, int64_t b) {
    const int64_t mats[7][2] = {{m, m}, {m, m}, {m, m}, {m, m}, {f, m}, {f, m}, {m, f}};
    int64_t total = 0;
    for (auto& a : mats) total += 2 * b * a[0] * a[1];  // Fprop
    if (!approx) {
        for (auto& a : mats) total += 2 * (2 * b * a[0] * a[1]);  // Wgrad + Dgrad
        return total;
    }
    for (int q = 4; q < 7; ++q) {
        const int64_t a = mats[q][0], c = mats[q][1], re = std::min(r, c);
        total += 2 * b * a * c * 2;                          // Rcomp + Dgrad
        total += 2 * re * (b * c + b * a + a * c);           // projected Wgrad
        total += svd_flops(a, c, re) / tau;                  // amortised SVD
    }
    return total;
}

}  // namespace

extern "C" {

int mecefo_cluster_create(mecefo_cluster** out, const mecefo_cluster_config* cfg) {
    if (!out || !cfg || cfg->dp < 1 || cfg->pp < 1 || cfg->layers < cfg->pp) return MECEFO_CTL_CONTRACT;
    if (cfg->kind < 0 || cfg->kind > 2 || cfg->recovery_iterations < 1) return MECEFO_CTL_CONTRACT;
    auto* c = new (std::nothrow) mecefo_cluster();
    if (!c) return MECEFO_CTL_CONTRACT;
    c->dp = cfg->dp;
    c->pp = cfg->pp;
    c->layers = cfg->layers;
    c->bounds.resize(cfg->pp + 1);
    for (int32_t s = 0; s <= cfg->pp; ++s)  // round(s * L / pp), Python round-half-even (cluster.py:59-62)
        c->bounds[s] = cfg->stage_boundaries ? cfg->stage_boundaries[s]
                                             : (int32_t)std::nearbyint((double)s * cfg->layers / cfg->pp);
    c->kind = cfg->kind;
    c->probability = cfg->probability;
    c->recovery_iterations = cfg->recovery_iterations;
    c->failure_interval_s = cfg->failure_interval_s;
    c->recovery_time_s = cfg->recovery_time_s;
    c->victim.assign((size_t)cfg->dp * cfg->pp, 0);
    c->has_victims = cfg->victims != nullptr;
    for (int32_t v = 0; c->has_victims && v < cfg->n_victims; ++v) {
        const int32_t i = cfg->victims[2 * v], s = cfg->victims[2 * v + 1];
        if (i >= 0 && i < cfg->dp && s >= 0 && s < cfg->pp) c->victim[(size_t)i * cfg->pp + s] = 1;
    }
    const uint64_t seed = cfg->seed;
    mecefo_pcg64_seed(&c->rng, &seed, 1);
    c->st.assign((size_t)cfg->dp * cfg->pp, 0);
    c->ex.resize((size_t)cfg->dp * cfg->pp);
    for (int32_t i = 0; i < cfg->dp; ++i)
        for (int32_t s = 0; s < cfg->pp; ++s) c->ex[(size_t)i * cfg->pp + s] = s;
    c->next_failure_time = cfg->failure_interval_s;
    *out = c;
    return MECEFO_CTL_OK;
}

int mecefo_cluster_destroy(mecefo_cluster* c) {
    delete c;
    return MECEFO_CTL_OK;
}

int mecefo_cluster_arrays(mecefo_cluster* c, int8_t** status, int32_t** executor) {
    if (!c || !status || !executor) return MECEFO_CTL_CONTRACT;
    *status = c->st.data();
    *executor = c->ex.data();
    return MECEFO_CTL_OK;
}

int mecefo_cluster_rng(mecefo_cluster* c, mecefo_pcg64_t** rng) {
    if (!c || !rng) return MECEFO_CTL_CONTRACT;
    *rng = &c->rng;
    return MECEFO_CTL_OK;
}

int mecefo_cluster_next_failure_time(mecefo_cluster* c, const double* set, double* get) {
    if (!c) return MECEFO_CTL_CONTRACT;
    if (set) c->next_failure_time = *set;
    if (get) *get = c->next_failure_time;
    return MECEFO_CTL_OK;
}

int mecefo_cluster_down_until(mecefo_cluster* c, int32_t* nodes, double* until, int32_t cap, int32_t* n) {
    if (!c || !n) return MECEFO_CTL_CONTRACT;
    *n = (int32_t)c->down_until.size();
    int32_t k = 0;
    for (auto& kv : c->down_until) {
        if (k >= cap) break;
        if (nodes) { nodes[2 * k] = kv.first / c->pp; nodes[2 * k + 1] = kv.first % c->pp; }
        if (until) until[k] = kv.second;
        ++k;
    }
    return MECEFO_CTL_OK;
}

int mecefo_cluster_set_down_until(mecefo_cluster* c, int32_t i, int32_t s, const double* until) {
    if (!c || i < 0 || i >= c->dp || s < 0 || s >= c->pp) return MECEFO_CTL_CONTRACT;
    if (until) c->down_until[i * c->pp + s] = *until;
    else c->down_until.erase(i * c->pp + s);
    return MECEFO_CTL_OK;
}

int mecefo_cluster_inject(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                          int32_t cap, int32_t* n) {
    if (!c || !n) return MECEFO_CTL_CONTRACT;
    EventSink ev{events, cap, 0};
    const int rc = inject(c, sim_time, iteration, ev);
    *n = ev.n;
    return rc;
}

int mecefo_cluster_due_recoveries(mecefo_cluster* c, double sim_time, int32_t iteration, int32_t* nodes,
                                  int32_t cap, int32_t* n) {
    if (!c || !n) return MECEFO_CTL_CONTRACT;
    const double clock = c->kind == 1 ? (double)iteration : sim_time;
    int32_t k = 0;
    for (auto& kv : c->down_until)  // std::map: ascending node index == sorted (i, s)
        if (clock >= kv.second) {
            if (k < cap && nodes) { nodes[2 * k] = kv.first / c->pp; nodes[2 * k + 1] = kv.first % c->pp; }
            ++k;
        }
    *n = k;
    return MECEFO_CTL_OK;
}

int mecefo_cluster_recover(mecefo_cluster* c, int32_t i, int32_t s, double sim_time, int32_t iteration,
                           mecefo_cluster_event* events, int32_t cap, int32_t* n) {
    if (!c || !n || i < 0 || i >= c->dp || s < 0 || s >= c->pp) return MECEFO_CTL_CONTRACT;
    EventSink ev{events, cap, 0};
    const int rc = recover(c, i, s, sim_time, iteration, ev);
    *n = ev.n;
    return rc;
}

int mecefo_cluster_reassign(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                            int32_t cap, int32_t* n) {
    if (!c || !n) return MECEFO_CTL_CONTRACT;
    EventSink ev{events, cap, 0};
    const int rc = reassign(c, sim_time, iteration, ev);
    *n = ev.n;
    return rc;
}

int mecefo_cluster_validate(const mecefo_cluster* c) { return c ? validate(c) : MECEFO_CTL_CONTRACT; }

int mecefo_cluster_step(mecefo_cluster* c, double sim_time, int32_t iteration, mecefo_cluster_event* events,
                        int32_t cap, int32_t* n) {
    if (!c || !n) return MECEFO_CTL_CONTRACT;
    EventSink ev{events, cap, 0};
    const double clock = c->kind == 1 ? (double)iteration : sim_time;
    std::vector<int32_t> due;
    for (auto& kv : c->down_until)
        if (clock >= kv.second) due.push_back(kv.first);
    int rc = MECEFO_CTL_OK;
    for (int32_t node : due)
        if ((rc = recover(c, node / c->pp, node % c->pp, sim_time, iteration, ev))) break;
    if (!rc) rc = inject(c, sim_time, iteration, ev);
    if (!rc) rc = reassign(c, sim_time, iteration, ev);
    if (!rc) rc = validate(c);
    *n = ev.n;
    return rc;
}

int mecefo_iteration_cost(const mecefo_cluster* c, int64_t hidden, int64_t ffn, int32_t policy_approx, int64_t r,
                          int64_t tau, int64_t tokens, int64_t* worst, int32_t* worst_stage, int64_t* total) {
    if (!c || !worst || !worst_stage || !total || tau < 1) return MECEFO_CTL_CONTRACT;
    const int64_t std_f = block_flops(hidden, ffn, 0, r, tau, tokens);
    const int64_t dbl_f = block_flops(hidden, ffn, policy_approx ? 1 : 0, r, tau, tokens);
    *worst = 0;
    *worst_stage = 0;
    *total = 0;
    for (int32_t i = 0; i < c->dp; ++i)
        for (int32_t node = 0; node < c->pp; ++node) {
            int64_t layers = 0;
            int32_t first = -1;
            for (int32_t s = 0; s < c->pp; ++s)
                if (c->ex[i * c->pp + s] == node) {
                    layers += c->bounds[s + 1] - c->bounds[s];
                    if (first < 0) first = s;
                }
            if (first < 0) continue;
            const int64_t fl = layers * (c->st[i * c->pp + node] == 0 ? std_f : dbl_f);
            *total += fl;
            if (fl > *worst) {
                *worst = fl;
                *worst_stage = first;
            }
        }
    return MECEFO_CTL_OK;
}

}  // extern "C"
