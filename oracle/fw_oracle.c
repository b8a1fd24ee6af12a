/*
 * fw_oracle.c -- CPU restatement of the reference parafw hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg load it, and only as the checker or as
 * the CPU arm.  It is pinned against the golden vectors in tests/golden/
 * (produced by the unmodified reference, tests/golden/make_golden.py).
 *
 * All citations are /root/reference/pkg/src/parafw/<file>:<line>.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define ORC_GAMMA 0x9E3779B97F4A7C15ULL

/* rng.py:31-35 -- one splitmix64 step */
uint64_t orc_splitmix64(uint64_t seed) {
    uint64_t z = seed + ORC_GAMMA;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.py:38-45 -- seeding (zero state replaced by the gamma) */
static uint64_t xs_seed(uint64_t seed) {
    uint64_t s = orc_splitmix64(seed);
    return s ? s : ORC_GAMMA;
}

/* rng.py:46-52 -- xorshift64* step */
static inline uint64_t xs_next(uint64_t *st) {
    uint64_t x = *st;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    *st = x;
    return x * 0x2545F4914F6CDD1DULL;
}

/* rng.py:54-62 -- bias-free bounded draw by rejection; n >= 1.
 * limit = 2^64 - (2^64 mod n); when n divides 2^64 nothing is rejected. */
static inline uint64_t xs_randbelow(uint64_t *st, uint64_t n) {
    uint64_t rem = (uint64_t)(-n) % n; /* == 2^64 mod n */
    if (rem == 0) return xs_next(st) % n;
    uint64_t limit = (uint64_t)0 - rem; /* 2^64 - rem */
    for (;;) {
        uint64_t r = xs_next(st);
        if (r < limit) return r % n;
    }
}

/* rng.py:70-76 -- chance(p): next_u64() < int(p * 2.0**64) */
static inline int xs_chance(uint64_t *st, double p) {
    if (p <= 0.0) return 0;
    if (p >= 1.0) return 1;
    double t = p * 18446744073709551616.0;
    uint64_t thr = (t >= 18446744073709551616.0) ? UINT64_MAX : (uint64_t)t;
    return xs_next(st) < thr;
}

/* rng.py:79-81 */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
    return orc_splitmix64(seed ^ orc_splitmix64(stream));
}

void orc_xs_stream(uint64_t seed, int64_t n, uint64_t *out) {
    uint64_t st = xs_seed(seed);
    for (int64_t i = 0; i < n; i++) out[i] = xs_next(&st);
}

/* traffic.py:117-130 (_draw_ip/_draw_packet) + traffic.py:158-160 (UNIFORM).
 * Draw order per packet: src_ip, src_port, dst_ip, dst_port. */
void orc_gen_traffic_uniform(uint64_t seed, int64_t n, int proto,
                             uint32_t src_base, int src_plen,
                             uint32_t dst_base, int dst_plen,
                             int sp_lo, int sp_hi, int dp_lo, int dp_hi,
                             uint8_t *o_proto, uint32_t *o_src, uint16_t *o_sport,
                             uint32_t *o_dst, uint16_t *o_dport) {
    uint64_t st = xs_seed(seed);
    uint64_t sspan = (uint64_t)1 << (32 - src_plen);
    uint64_t dspan = (uint64_t)1 << (32 - dst_plen);
    for (int64_t i = 0; i < n; i++) {
        o_proto[i] = (uint8_t)proto;
        o_src[i] = (uint32_t)(src_base + xs_randbelow(&st, sspan));
        o_sport[i] = (uint16_t)(sp_lo + xs_randbelow(&st, (uint64_t)(sp_hi - sp_lo + 1)));
        o_dst[i] = (uint32_t)(dst_base + xs_randbelow(&st, dspan));
        o_dport[i] = (uint16_t)(dp_lo + xs_randbelow(&st, (uint64_t)(dp_hi - dp_lo + 1)));
    }
}

/* model.py:108-114 -- prefix mask with the /0 special case */
static inline uint32_t cidr_mask(int plen) {
    return plen == 0 ? 0u : (uint32_t)(0xFFFFFFFFull << (32 - plen));
}

/* traffic.py:194-229 (generate_ruleset, _draw_cidr, _draw_ports) emitted in the
 * CompiledRuleset column form of classifier.py:120-134. */
void orc_gen_ruleset(int64_t count, uint64_t seed, double wp, double action_split,
                     uint8_t *proto, uint32_t *src_base, uint32_t *src_mask,
                     uint16_t *sport_lo, uint16_t *sport_hi,
                     uint32_t *dst_base, uint32_t *dst_mask,
                     uint16_t *dport_lo, uint16_t *dport_hi, uint8_t *accept) {
    static const uint8_t concrete[3] = {6, 17, 1}; /* traffic.py:63 TCP, UDP, ICMP */
    uint64_t st = xs_seed(seed);
    for (int64_t i = 0; i < count; i++) {
        accept[i] = (uint8_t)xs_chance(&st, action_split);
        if (xs_chance(&st, wp)) proto[i] = 0;
        else proto[i] = concrete[xs_randbelow(&st, 3)];
        for (int f = 0; f < 4; f++) {
            if (f == 0 || f == 2) { /* _draw_cidr, traffic.py:194-198 */
                uint32_t base = 0, mask = 0;
                if (!xs_chance(&st, wp)) {
                    int plen = 8 + (int)xs_randbelow(&st, 25);
                    uint32_t raw = (uint32_t)xs_randbelow(&st, (uint64_t)1 << 32);
                    mask = cidr_mask(plen);
                    base = raw & mask; /* model.py:106 normalisation */
                }
                if (f == 0) { src_base[i] = base; src_mask[i] = mask; }
                else { dst_base[i] = base; dst_mask[i] = mask; }
            } else { /* _draw_ports, traffic.py:201-206 */
                uint16_t lo = 0, hi = 65535;
                if (!xs_chance(&st, wp)) {
                    uint16_t a = (uint16_t)xs_randbelow(&st, 65536);
                    uint16_t b = (uint16_t)xs_randbelow(&st, 65536);
                    lo = a < b ? a : b;
                    hi = a < b ? b : a;
                }
                if (f == 1) { sport_lo[i] = lo; sport_hi[i] = hi; }
                else { dport_lo[i] = lo; dport_hi[i] = hi; }
            }
        }
    }
}

/* model.py:222-230 (rule_matches) in the integer form of classifier.py:136-144 */
static inline int rule_hit(int64_t r, const uint8_t *proto, const uint32_t *sb, const uint32_t *sm,
                           const uint16_t *slo, const uint16_t *shi, const uint32_t *db,
                           const uint32_t *dm, const uint16_t *dlo, const uint16_t *dhi,
                           uint8_t pp, uint32_t ps, uint16_t psp, uint32_t pd, uint16_t pdp) {
    return (proto[r] == 0 || proto[r] == pp) && ((ps & sm[r]) == sb[r]) &&
           (psp >= slo[r] && psp <= shi[r]) && ((pd & dm[r]) == db[r]) &&
           (pdp >= dlo[r] && pdp <= dhi[r]);
}

/* classifier.py:146-162 (scan_range): earliest matching index in [lo, hi) per
 * packet, or -1.  Restated as the per-packet early-exit loop of
 * classifier.py:54-59 (classify), which scan_range is equivalent to; packets
 * are independent, so they are split across threads in contiguous balanced
 * chunks exactly as the data-parallel model splits them (engines.py:143-154,
 * engines.py:302-314). */
typedef struct {
    const uint8_t *proto; const uint32_t *sb, *sm; const uint16_t *slo, *shi;
    const uint32_t *db, *dm; const uint16_t *dlo, *dhi;
    const uint8_t *pp; const uint32_t *ps; const uint16_t *psp; const uint32_t *pd;
    const uint16_t *pdp; int64_t lo, hi, p0, p1; int64_t *first;
} scan_job;

static void *scan_worker(void *arg) {
    const scan_job *j = (const scan_job *)arg;
    for (int64_t i = j->p0; i < j->p1; i++) {
        int64_t f = -1;
        for (int64_t r = j->lo; r < j->hi; r++) {
            if (rule_hit(r, j->proto, j->sb, j->sm, j->slo, j->shi, j->db, j->dm, j->dlo, j->dhi,
                         j->pp[i], j->ps[i], j->psp[i], j->pd[i], j->pdp[i])) {
                f = r;
                break;
            }
        }
        j->first[i] = f;
    }
    return NULL;
}

int orc_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

void orc_scan_range(const uint8_t *proto, const uint32_t *sb, const uint32_t *sm,
                    const uint16_t *slo, const uint16_t *shi, const uint32_t *db,
                    const uint32_t *dm, const uint16_t *dlo, const uint16_t *dhi,
                    int64_t n, const uint8_t *pp, const uint32_t *ps, const uint16_t *psp,
                    const uint32_t *pd, const uint16_t *pdp, int64_t lo, int64_t hi,
                    int64_t *first, int nthreads) {
    enum { MAXT = 512 };
    if (nthreads < 1) nthreads = orc_max_threads();
    if (nthreads > MAXT) nthreads = MAXT;
    if (n < nthreads) nthreads = n > 0 ? (int)n : 1;
    scan_job jobs[MAXT];
    pthread_t tid[MAXT];
    int64_t base = n / nthreads, extra = n % nthreads, p = 0;
    for (int t = 0; t < nthreads; t++) {
        int64_t q = p + base + (t < extra ? 1 : 0);
        jobs[t] = (scan_job){proto, sb, sm, slo, shi, db, dm, dlo, dhi, pp, ps, psp, pd, pdp,
                             lo, hi, p, q, first};
        p = q;
    }
    for (int t = 1; t < nthreads; t++) pthread_create(&tid[t], NULL, scan_worker, &jobs[t]);
    scan_worker(&jobs[0]);
    for (int t = 1; t < nthreads; t++) pthread_join(tid[t], NULL);
}
