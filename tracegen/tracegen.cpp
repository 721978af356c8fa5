// tracegen/tracegen.cpp -- seeded synthetic malloc/free trace generator.
//
// Input generator shared by the oracle tests and the CUDA path.  It holds
// none of the method's arithmetic (no footprint, sampler, tracker or
// scoring): it only emits valid event streams "shaped like Python
// workloads" (SURVEY.md §8(d) "Generator model"):
//   * site popularity: Zipf(s) over n_sites; the Zipf rank IS the site id
//     (ids are dense, hottest first -- the order in which a profiler's site
//     table would first see them);
//   * per-site size class: small pymalloc-like objects {16..512} B with short
//     geometric lifetimes (the "short-lived objects created by the Python
//     interpreter itself"), medium lognormal objects, and rare
//     NumPy-like array buffers with Pareto sizes;
//   * planted leak sites that allocate and never free;
//   * pointers from a 16-B aligned bump allocator with per-size LIFO reuse,
//     so freed addresses are reused (pointer identity matters).
// Every trace is valid by construction (reading Q16): each free matches a
// live prior alloc of the same size; live pointers are unique.
//
// Determinism: trace t of a config draws only from xoshiro256** seeded by
// splitmix64(config_seed ^ t), so any subset of traces can be regenerated
// independently (the bench and the tests regenerate the same bytes).
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <queue>
#include <thread>
#include <atomic>
#include <unordered_map>
#include <algorithm>

namespace {

inline uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t s[4];
    explicit Rng(uint64_t seed) { uint64_t x = seed; for (auto& v : s) v = splitmix64(x); }
    static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    inline uint64_t next() {
        uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
        return r;
    }
    inline double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }  // [0,1)
    inline double uniform_pos() { return ((double)(next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); } // (0,1)
    inline double normal() {  // Box-Muller
        double u1 = uniform_pos(), u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

enum SiteClass : uint8_t { SMALL = 0, MEDIUM = 1, ARRAY = 2, LEAK = 3 };

}  // namespace

extern "C" {

struct tg_config {
    uint32_t n_traces;
    uint32_t n_sites;
    uint64_t events_per_trace;
    double   zipf_s;
    uint32_t n_planted;        // planted leak sites
    uint32_t heavy_tailed;     // config 5: alpha 1.1, cap 4 GiB, 5% array sites
    uint64_t leak_T;           // threshold the planted leak sizes are scaled to: U[T/4, T]
    double   leak_lambda;      // per-step probability of a planted-leak allocation
    double   leak_rate_spread; // planted site k drawn with weight spread^(k/(n-1)) (config 3: 100)
    uint64_t seed;             // config seed, 20221215 + cfg
    double   copy_lambda;      // per-step probability of a copy event (kind 2); 0: none
};

struct tg_event { uint64_t ptr; uint64_t meta; };

}  // extern "C"

namespace {

constexpr uint64_t SMALL_BASE = 0x0000100000000000ull;
constexpr uint64_t LARGE_BASE = 0x00007f0000000000ull;

inline uint64_t pack(uint64_t size, unsigned kind, uint32_t site) {
    return (size & ((1ull << 40) - 1)) | ((uint64_t)kind << 40) | ((uint64_t)site << 43);
}

struct Model {
    tg_config c;
    std::vector<double> zipf_cdf;      // over ranks 0..n_sites-1
    std::vector<uint8_t> cls;          // per site
    std::vector<double> life_mean;     // per site (events)
    std::vector<uint32_t> planted;     // planted site ids
    std::vector<double> planted_cdf;   // selection weights among planted sites
    double alpha, arr_cap;

    explicit Model(const tg_config& cfg) : c(cfg) {
        uint32_t S = c.n_sites;
        zipf_cdf.resize(S);
        double acc = 0;
        for (uint32_t r = 0; r < S; ++r) { acc += 1.0 / std::pow((double)(r + 1), c.zipf_s); zipf_cdf[r] = acc; }
        for (auto& v : zipf_cdf) v /= acc;
        zipf_cdf[S - 1] = 1.0;
        cls.resize(S); life_mean.resize(S);
        uint64_t x = c.seed ^ 0x5173000000000000ull;
        double p_small = c.heavy_tailed ? 0.80 : 0.85, p_med = c.heavy_tailed ? 0.95 : 0.99;
        for (uint32_t s = 0; s < S; ++s) {
            double u = (double)(splitmix64(x) >> 11) * (1.0 / 9007199254740992.0);
            double v = (double)(splitmix64(x) >> 11) * (1.0 / 9007199254740992.0);
            if (u < p_small)     { cls[s] = SMALL;  life_mean[s] = 16.0; }
            else if (u < p_med)  { cls[s] = MEDIUM; life_mean[s] = 1000.0; }
            else                 { cls[s] = ARRAY;  life_mean[s] = std::pow(10.0, 4.0 + v); }
        }
        // planted leak sites: spread over the colder half of the ranks
        for (uint32_t k = 0; k < c.n_planted && k < S; ++k) {
            uint32_t s = S - 1 - (uint32_t)(((uint64_t)k * (S / 2)) / std::max<uint32_t>(c.n_planted, 1));
            cls[s] = LEAK; planted.push_back(s);
        }
        double pacc = 0;
        for (uint32_t k = 0; k < planted.size(); ++k) {
            double w = planted.size() > 1 && c.leak_rate_spread > 0
                ? std::pow(c.leak_rate_spread, (double)k / (double)(planted.size() - 1)) : 1.0;
            pacc += w; planted_cdf.push_back(pacc);
        }
        for (auto& v : planted_cdf) v /= pacc;
        alpha = c.heavy_tailed ? 1.1 : 1.2;
        arr_cap = c.heavy_tailed ? 4294967296.0 : 1073741824.0;
    }

    uint32_t zipf(Rng& g) const {
        double u = g.uniform();
        return (uint32_t)(std::lower_bound(zipf_cdf.begin(), zipf_cdf.end(), u) - zipf_cdf.begin());
    }

    uint64_t size_for(uint32_t s, Rng& g) const {
        switch (cls[s]) {
        case SMALL:  return 16ull * (1 + (g.next() >> 59));                          // {16,...,512}
        case MEDIUM: {
            double v = 4096.0 * std::exp(1.0 * g.normal());
            if (v > 1048576.0) v = 1048576.0;
            if (v < 16.0) v = 16.0;
            return ((uint64_t)v + 15) & ~15ull;
        }
        case ARRAY: {
            double v = 65536.0 / std::pow(g.uniform_pos(), 1.0 / alpha);              // Pareto(x_min=64Ki)
            if (v > arr_cap) v = arr_cap;
            return ((uint64_t)v + 15) & ~15ull;
        }
        default: {                                                                     // planted leak
            uint64_t lo = std::max<uint64_t>(c.leak_T / 4, 16), hi = std::max<uint64_t>(c.leak_T, lo);
            return lo + (g.next() % (hi - lo + 1));
        }
        }
    }

    uint64_t lifetime(uint32_t s, Rng& g) const {
        double l = -life_mean[s] * std::log(g.uniform_pos());                        // geometric ~ exponential
        return 1 + (uint64_t)l;
    }

    void gen_trace(uint32_t t, tg_event* out) const {
        uint64_t x = c.seed ^ (uint64_t)t;
        Rng g(splitmix64(x));
        const uint64_t n = c.events_per_trace;
        struct Live { uint64_t death; uint64_t ptr; uint64_t size; };
        auto cmp = [](const Live& a, const Live& b) { return a.death > b.death; };
        std::priority_queue<Live, std::vector<Live>, decltype(cmp)> heap(cmp);
        std::vector<std::vector<uint64_t>> small_free(33);
        std::unordered_map<uint64_t, std::vector<uint64_t>> large_free;
        uint64_t small_bump = SMALL_BASE, large_bump = LARGE_BASE;
        for (uint64_t i = 0; i < n; ++i) {
            if (!heap.empty() && heap.top().death <= i) {                            // a due free
                Live o = heap.top(); heap.pop();
                out[i].ptr = o.ptr;
                out[i].meta = pack(o.size, 1, zipf(g));                                // free site = current line
                if (o.size <= 512) small_free[o.size >> 4].push_back(o.ptr);
                else large_free[o.size].push_back(o.ptr);
                continue;
            }
            if (c.copy_lambda > 0 && g.uniform() < c.copy_lambda) {                 // a memcpy at the current
                const uint32_t cs = zipf(g);                                          // line, of an object-sized
                out[i].ptr = 0;                                                       // buffer (no draw at all
                out[i].meta = pack(size_for(cs, g), 2, cs);                           // when copy_lambda == 0)
                continue;
            }
            uint32_t s;
            bool leak = false;
            if (!planted.empty() && g.uniform() < c.leak_lambda) {
                double u = g.uniform();
                s = planted[std::lower_bound(planted_cdf.begin(), planted_cdf.end(), u) - planted_cdf.begin()];
                leak = true;
            } else {
                do { s = zipf(g); } while (cls[s] == LEAK);                           // leaks only via lambda
            }
            uint64_t size = size_for(s, g);
            uint64_t p;
            if (size <= 512) {
                auto& fl = small_free[size >> 4];
                if (!fl.empty()) { p = fl.back(); fl.pop_back(); }
                else { p = small_bump; small_bump += size; }
            } else {
                auto it = large_free.find(size);
                if (it != large_free.end() && !it->second.empty()) { p = it->second.back(); it->second.pop_back(); }
                else { p = large_bump; large_bump += (size + 4095) & ~4095ull; }
            }
            out[i].ptr = p;
            out[i].meta = pack(size, 0, s) | (cls[s] == SMALL ? (1ull << 42) : 0ull);  // domain: small objects are
                                                                                    // the interpreter's (managed)
            if (!leak) heap.push(Live{i + lifetime(s, g), p, size});
        }
    }
};

}  // namespace

extern "C" {

// Generate traces [t0, t1) of the config into out (events_per_trace each,
// trace t0 first), on n_threads threads.  Returns 0.
int tg_generate(const tg_config* cfg, uint32_t t0, uint32_t t1, tg_event* out, int n_threads) {
    Model m(*cfg);
    std::atomic<uint32_t> next{t0};
    auto work = [&]() {
        for (;;) {
            uint32_t t = next.fetch_add(1);
            if (t >= t1) break;
            m.gen_trace(t, out + (uint64_t)(t - t0) * cfg->events_per_trace);
        }
    };
    if (n_threads < 1) n_threads = 1;
    std::vector<std::thread> th;
    for (int k = 1; k < n_threads; ++k) th.emplace_back(work);
    work();
    for (auto& x : th) x.join();
    return 0;
}

// Per-site class (0 small, 1 medium, 2 array, 3 planted leak) -> out[n_sites].
int tg_site_classes(const tg_config* cfg, uint8_t* out) {
    Model m(*cfg);
    std::memcpy(out, m.cls.data(), cfg->n_sites);
    return 0;
}

}  // extern "C"
