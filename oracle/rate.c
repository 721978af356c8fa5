/*
 * oracle/rate.c -- CPU ORACLE FOR THE RATE-BASED BYTE SAMPLER.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the product never links or calls it.
 *
 * P:414-427 (sec:memory-sampling): "each byte allocated or freed corresponds to a Bernoulli
 * trial with a given probability p of sampling ... these samplers initialize counters to random
 * numbers drawn from a Poisson process or a geometric distribution with the same parameter. Each
 * allocation and free then decrements this counter by the number of bytes allocated and freed,
 * and triggers a sample when the counter drops below 0."  SPEC rate-sampler: the
 * counter is re-drawn after a sample and the draw is added to the residual, so one large event
 * can trigger several samples; geometric draws; a deterministic mode (counter = R,
 * S:178) for tests.  P:500-518 / S:410-413: copy volume uses the same sampler on copied bytes.
 *
 * Readings: "drops below 0" is strict (counter < 0); draw k of trace t comes from
 * a counter-based generator keyed by (seed, t, k); seed 0 is the deterministic mode; the counted
 * event kinds are a mask (alloc|free for the baseline, copy for copy volume).
 *
 * The geometric draw G = 1 + floor(ln u / ln(1 - 1/R)), u in (0, 1], uses the fixed-order
 * logarithm below (no library log, no FMA: -ffp-contract=off) so that it is exactly
 * reproducible; ln is pinned against the C library's log in tests/test_oracle_rate.py.
 */
#include <math.h>
#include <stdint.h>
#include "oracle.h"

/* ln x for x > 0: x = m 2^e with m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh(f), f = (m-1)/(m+1),
 * atanh(f) = f (1 + f^2/3 + f^4/5 + ... + f^22/23), Horner from the highest term. */
double orc_soft_log(double x)
{
    static const double c[12] = {
        0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
        0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
        0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5 };
    int e = 0;
    double m = frexp(x, &e);                 /* m in [0.5, 1) */
    if (m < 0x1.6a09e667f3bcdp-1) { m = m * 2.0; e -= 1; }
    const double f = (m - 1.0) / (m + 1.0);
    const double f2 = f * f;
    double s = c[11];
    for (int j = 10; j >= 0; --j) { s = s * f2; s = s + c[j]; }
    const double r = (2.0 * f) * s;
    return r + (double)e * 0x1.62e42fefa39efp-1;
}

static uint64_t splitmix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Draw k >= 1 of trace t: the countdown reload (a geometric variate with mean R). */
uint64_t orc_rate_draw(uint64_t R, uint64_t seed, uint32_t trace, uint64_t k)
{
    if (seed == 0) return R;                                 /* deterministic mode */
    if (R <= 1) return 1;                                    /* p = 1: every byte is a trial success */
    const uint64_t x = splitmix64(seed ^ splitmix64(((uint64_t)trace << 40) ^ k));
    const double u = (double)((x >> 11) + 1) * 0x1.0p-53;    /* (0, 1] */
    const double lq = orc_soft_log(1.0 - 1.0 / (double)R);   /* ln(1 - p) < 0 */
    const double g = floor(orc_soft_log(u) / lq);
    return (uint64_t)g + 1;
}

/* One trace, in event order: counter = draw 1; each counted event subtracts its
 * size; while the counter is below 0, a sample (event index, cumulative draws S_k, site, kind)
 * and the next draw is added.  Returns 0, or -1 for an invalid event kind 3. */
int orc_rate_trace(const orc_event* ev, uint64_t n, uint64_t R, uint64_t seed, uint32_t trace,
                   unsigned kinds, orc_rate_sample* out, uint64_t cap, uint64_t* n_samples)
{
    uint64_t k = 1;
    uint64_t S = orc_rate_draw(R, seed, trace, 1);           /* S_k = G_1 + ... + G_k */
    int64_t C = (int64_t)S;
    uint64_t ns = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const unsigned kind = (unsigned)(ev[i].meta >> 40) & 3u;
        if (kind == 3) return -1;
        if (!((kinds >> kind) & 1u)) continue;
        C -= (int64_t)(ev[i].meta & ((1ull << 40) - 1));
        while (C < 0) {
            if (ns < cap) {
                orc_rate_sample* s = &out[ns];
                s->idx = i; s->draw_sum = S; s->site = (uint32_t)(ev[i].meta >> 43); s->kind = kind;
            }
            ++ns; ++k;
            const uint64_t g = orc_rate_draw(R, seed, trace, k);
            S += g; C += (int64_t)g;
        }
    }
    *n_samples = ns;
    return 0;
}
