// pfw.cu -- B200 (sm_100a) packet-filter hot path behind the C-ABI of include/pfw.h.
//
// Reference semantics (parafw, /root/reference/pkg/src/parafw):
//   rule predicate            model.py:222-230, classifier.py:136-144
//   first-match in [lo,hi)    classifier.py:146-162
//   comparison accounting     classifier.py:200, engines.py:312, engines.py:366-368
//   min-combine               engines.py:202-212
//   traffic generator         rng.py:31-62, traffic.py:117-130, 148-160
//
// Design (DESIGN.md has the full rationale and rooflines):
//   * every rule field is a range test  (x - lo) <=u width  on 32-bit lanes:
//       src/dst CIDR  -> lo = base, width = ~mask      (x & mask) == base
//       ports         -> lo = lo,   width = hi - lo    lo <= x <= hi
//       proto         -> ANY: width = ~0; else lo = proto, width = 0
//     one IMAD (FMA pipe, "x*1 + (-lo)") + one ISETP (ALU pipe) per field, so
//     a 5-field rule test is 10 integer ops split evenly over the two pipes.
//   * packet x rule grid: a CTA owns a tile of packets in shared memory; all
//     of its warps hold the same 32*KS-rule stage in registers (lane l holds
//     rules stage+32j+l, j < KS) and split the tile's LIVE packets.  Per packet
//     each lane evaluates its KS rules, one __any_sync decides whether the
//     stage hit, and __ballot_sync/__ffs over the sub-chunks in order yields
//     the lowest matching index.  Stages run in rule order and matched packets
//     retire from the live list after every stage, so no packet is tested
//     past the stage that holds its first match (early exit at 32*KS rules).
//   * stage rules are TMA-bulk-copied (cp.async.bulk + mbarrier) into a
//     double-buffered shared-memory ring while the previous stage computes.
//   * persistent grid (SMs x resident CTAs), tiles handed out by an atomic
//     counter (dynamic load balance: tiles differ in work by >10x).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>
#include <mutex>
#include <string>
#include <vector>
#include <atomic>
#include <algorithm>
#include <type_traits>

#include "../../include/pfw.h"
#include <nvtx3/nvToolsExt.h>
#include "hostpool.h"
#include <chrono>  // header-only NVTX v3: ranges cost nothing unless a tool is attached

#define PFW_VERSION "0.2.0"

// -DPFW_CHECKS builds device-side bounds assertions into every derived index
// (compute-sanitizer is not available on the GPU pool): a violated check
// traps the kernel, which the parity suite then reports as a CUDA error.
#ifdef PFW_CHECKS
#define PFW_CHECK(cond) \
    do {                \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define PFW_CHECK(cond) \
    do {                \
    } while (0)
#endif

namespace {

// ------------------------------------------------------------------ errors
thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int set_err(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// NVTX range for the lifetime of a scope (pack / upload / scan / e2e stages)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e__ = (expr);                                                        \
        if (e__ != cudaSuccess)                                                          \
            return set_err(PFW_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e__), \
                           __FILE__, __LINE__);                                          \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// ---------------------------------------------------------- rule encoding
// Device rule table: SoA of NF words, field f of rule r at rules[f * rpad + r].
constexpr int NF = 10;
// Per rule (one register each when staged):
//   IP fields, 32-bit integer range tests on the FMA-heavy + ALU pipes:
//     F_SRC_NLO = -src_base, F_SRC_W = ~src_mask  ->  (src - base) <=u ~mask
//   port/proto fields, fp32 range tests on exact integers < 2^24 (FFMA runs on
//   both FMA halves), the protocol folded into the port words:
//     packet A  = (proto << 16) | sport   proto-major: concrete-proto rules
//     packet A2 = (sport << 8)  | proto   proto-minor: ANY-proto rules
//     packet B  = (dport << 8)  | proto   proto-minor: every rule
//     dA = (A - A2)*c1 + (A2 - loA) with c1 = 1 concrete, 0 ANY (A - A2 is
//     precomputed per packet; F_A_C2 = 1 - c1 stays in the table, unused);
//     dB = B - loB; a field matches iff 0 <= d <= w, tested as
//     float_bits(d) <=u float_bits(w) (negative d has the sign bit set).
enum { F_SRC_NLO = 0, F_SRC_W, F_DST_NLO, F_DST_W, F_A_C1, F_A_C2, F_A_NLO, F_A_W, F_B_NLO,
       F_B_W };
constexpr uint32_t NEVER_B_NLO = 0x4C000000u;  // +2^25: dB >= 2^25 > any width (< 2^24)
constexpr uint32_t NEVER_B_W = 0u;             // +0.0f

// Tunables (pfw_set_tuning)
int g_ks = 8;            // rules per lane per stage (stage = 32*KS rules)
int g_tile = 2048;       // packets per CTA tile
int g_ctas_per_sm = 0;   // 0 = occupancy query
int g_force_imad = 1;    // route the subtract through IMAD (FMA pipe)
int g_first_pass = 1024; // rules in the first pass (0 = single pass); passes double
constexpr int MAX_PASSES = 32;
constexpr int MAX_PEERS = 64;
constexpr int E2E_SLOTS = 3;
constexpr int64_t E2E_SMALL = 4096;  // host batches up to this size take the packed one-copy path
constexpr int MAX_CHAINS = 257;
int g_proto_split = 0;   // opt-in: scan protocol-split rule chains
int g_short_circuit = 0; // warp-level short-circuit of the port tests (SC variant; measured slower)
int g_bucket = 1;        // group large batches by protocol (protocol-uniform tiles)
int64_t g_bucket_min = 1 << 20;  // ... from this many packets on

}  // namespace

// Per-scan scratch: ping-pong live-id lists for the passes + counters, and
// the protocol buckets of launch_split.  Scans that may run concurrently
// (the e2e pipeline's two compute streams) each get their own.
struct ScanWs {
    uint32_t *ids = nullptr;       // 2 * cap
    unsigned int *ctr = nullptr;   // 2 * MAX_PASSES
    int64_t cap = 0;
    uint32_t *d_bucket = nullptr;  // packet ids grouped by chain (bucket_cap)
    unsigned *d_bcount = nullptr;  // [3 * MAX_CHAINS + 1]: count, base, cursor, single flag
    int64_t bucket_cap = 0;
};

// Per-field match sets (matchset.cuh): field value -> elementary interval ->
// bitmap row of the rules whose test on that field holds there.
struct MatchSet {
    int64_t wp = 0;             // 32-bit words per bitmap row (whole 128-byte lines)
    int64_t rows[4] = {};       // rows of src, dst, (protocol class, sport), dport
    uint32_t *d_bits_all = nullptr;  // the four dimensions' rows, one allocation
    uint32_t *d_bits[4] = {};   // rows[d] * wp words each (inside d_bits_all)
    uint32_t *d_ipb[2] = {};    // src / dst interval boundaries (sorted, [0] = 0)
    uint4 *d_ipc[2] = {};       // per /16 block: first boundary index | count << 24, 6 boundary low halves
    uint16_t *d_port[2] = {};   // sport / dport -> interval (65536 entries each)
    uint32_t *d_pbk[2] = {};    // the same as 2048 buckets of 32 ports (12 KB: boundary bits, then u16 bases)
    uint8_t *d_cls = nullptr;   // protocol -> class (256 entries)
    int64_t sp_rows = 0;        // sport intervals = rows per protocol class
    size_t bytes = 0;           // device bytes of all of the above
    // summaries: bit k of a row's summary = block k (1024 rules) of the row non-zero
    uint32_t *d_sum[4] = {};
    int64_t sw = 0;             // summary words per row (0: not built)
    double sum_keep = 1.0;      // expected fraction of blocks a packet's AND-summary keeps
    bool use_sum = false;       // scan with summaries (auto: sum_keep below the threshold)
    // compressed rows (large rulesets): inside one 1024-rule block, rows differ
    // only where a boundary of that block's rules separates them, so each
    // (dimension, block) stores its <= 2*1024+1 distinct 128-byte lines once and
    // each row a u16 line index per block; the plain rows are then dropped
    bool cmp = false;
    int64_t nblk = 0;           // blocks per row (wp / 32)
    int64_t pstride = 0;        // u16 entries per row of line indices (>= nblk + 16, multiple of 8)
    uint16_t *d_ptr_all = nullptr;  // line indices: dimension d's rows at ptr_off[d]
    uint64_t ptr_off[4] = {};
    uint32_t *d_lines = nullptr;    // distinct lines, 32 words each
    uint32_t *d_loff = nullptr;     // [4 * nblk]: first line of (d, block)
    int64_t nlines = 0;
    uint16_t *d_head_all = nullptr; // rows x 8: the first 8 blocks' line indices, dense (L2-resident)
    uint64_t head_off[4] = {};
};

struct pfw_ruleset {
    int device;
    int64_t n;       // rules
    int64_t index_base = 0;  // rule shard: these are rules [index_base, index_base + n) of total
    int64_t total = -1;      // size of the whole ruleset (-1: this handle is the whole ruleset)
    int64_t rpad;    // padded row length (multiple of 32, >= n + max stage)
    uint32_t *d_rules = nullptr;   // NF * rpad
    uint8_t *d_accept = nullptr;   // rpad
    int sms = 148;
    // e2e workspace
    void *d_ws = nullptr;
    size_t ws_bytes = 0;
    void *h_stage = nullptr;       // pinned staging ring for pageable e2e buffers (same slots as d_ws)
    size_t stage_bytes = 0;
    void *h_small = nullptr;       // pinned buffer of the packed tiny-batch path (E2E_SMALL packets)
    cudaStream_t streams[4] = {};  // e2e copy-in, compute x2 (alternating chunks), copy-out
    cudaEvent_t events[3 * 3] = {};                          // e2e per-slot in / scan / out
    ScanWs ws;         // default (calls on the caller's stream)
    uint32_t **d_peers = nullptr;  // 2 * MAX_PEERS device pointer table (fused combine)
    ScanWs ws_e2e[2];  // pfw_classify_host slots
    // Protocol-split rule chains (opt-in, tuning "proto_split"): chain c holds,
    // in rule order, the rules a packet of protocol proto_of[c] can match
    // (proto == that value or ANY); the last chain holds only the ANY rules
    // (packets whose protocol no rule names).  lut[p] = chain of protocol p.
    struct Chain {
        int64_t n = 0, rpad = 0;
        uint32_t *d_rules = nullptr;  // NF * rpad, same encoding as d_rules
        uint32_t *d_orig = nullptr;   // chain position -> original rule index
        std::vector<uint32_t> orig;
    };
    std::vector<Chain> chains;
    uint8_t *d_lut = nullptr;          // 256 entries
    MatchSet *ms = nullptr;            // match sets (null: not built / over budget)
};

namespace {


// ================================================================ kernels

// The reference's own packet layout (PacketArrays, classifier.py:62-95): five
// SoA columns, 13 bytes per packet.  Scans read either these or 16-byte records.
struct PacketCols {
    const uint8_t *proto;
    const uint32_t *src;
    const uint16_t *sport;
    const uint32_t *dst;
    const uint16_t *dport;
};

struct ScanParams {
    const uint32_t *rules;
    const uint8_t *accept;
    int64_t rpad;
    int64_t lo, hi;            // rule window [lo, hi) in table positions (masking, stages)
    int64_t win_lo, win_hi;    // the same window in original rule indices (comparisons)
    const uint32_t *orig;      // table position -> original rule index (null = identity)
    int chain;                 // table is a protocol-split chain (protocol-free encoding)
    int64_t s_begin, s_end;    // this pass: stage starts s_begin, s_begin+STAGE, ... < s_end
    const uint4 *pkts;         // 16-byte records, or null: read the columns in `cols`
    PacketCols cols;
    int64_t n;                 // packets in the batch (pass 0 count when in_ids == null)
    const uint32_t *in_ids;    // live packet ids of this pass (null = 0..n-1)
    const unsigned int *in_count;  // device count of in_ids (null = n)
    const unsigned int *bucket_base;  // pass 0 of a chain scan: in_ids offset (device)
    const int *bk_single;             // pass 0 of a bucketed scan: only non-empty bucket, or -1
    int bk_index;                     // this launch's bucket
    const uint32_t *in_ids0;          // pass-0 input of a launch (null = identity)
    const unsigned int *in_count0;
    uint32_t *out_ids;         // survivors of this pass (null = final pass)
    unsigned int *out_count;
    int64_t out_cap;           // capacity of out_ids (checks)
    uint32_t *first;
    uint32_t *comps;
    uint8_t *verdict;
    unsigned long long *stats;
    unsigned int *tile_counter;
    unsigned long long *blocks_read;  // match-set scan with summaries: block reads (null = not counted)
    int tile;
    uint32_t one;  // runtime 1: keeps ptxas from folding x*1+c into IADD3
    uint32_t nomatch_out;  // MODE_WRITE: first[] value of an unmatched packet (PFW_NO_MATCH, or -1 for host views)
    uint32_t index_base;  // rule shard: reported indices are index_base + local position
    // MODE_PEER (fused function-parallel combine): result buffers of every
    // rank, reached over NVLink through CUDA IPC mappings
    uint32_t *const *peer_first;
    uint32_t *const *peer_comps;
    int npeers;
    int scatter;  // 1: packet id lives on its owner rank (balanced shards of n)
};

enum { MODE_WRITE = 0, MODE_ACC = 1, MODE_PEER = 2 };

// Result epilogue shared by the scan kernels: packet `id` first matches
// original rule f (or PFW_NO_MATCH) inside the window; writes first /
// comparisons / verdict (MODE_WRITE), accumulates a function-parallel
// partition (MODE_ACC), or combines straight into the ranks' buffers
// (MODE_PEER); span = window length (comparisons of an unmatched packet).
template <int MODE, bool CS = false>
__device__ __forceinline__ void emit_result(const ScanParams &p, uint32_t id, uint32_t f, uint32_t span,
                                            unsigned long long &st_sum, unsigned &st_max) {
    const uint32_t c = (f != PFW_NO_MATCH) ? (uint32_t)(f - p.win_lo + 1) : span;
    const uint32_t fl = f;  // local position (actions)
    if (f != PFW_NO_MATCH) f += p.index_base;  // reported index (rule shards: global)
    if (MODE == MODE_ACC) {
        if (f != PFW_NO_MATCH) p.first[id] = min(p.first[id], f);
        p.comps[id] += c;
    } else if (MODE == MODE_PEER) {
        // the engines.py:202-212 min-combine and :366-367 sum, issued straight
        // from the scan epilogue into the ranks' buffers (NVLink atomics),
        // overlapping the transfer with the remaining tiles' compute
        if (p.scatter) {
            const uint64_t q = (uint64_t)p.n / (uint64_t)p.npeers;
            const uint64_t r = (uint64_t)p.n % (uint64_t)p.npeers;
            const uint64_t big = (q + 1) * r;
            const uint64_t o = id < big ? id / (q + 1) : r + (id - big) / q;
            const uint64_t off = id - (o < r ? o * (q + 1) : big + (o - r) * q);
            PFW_CHECK(o < (uint64_t)p.npeers && off < (o < r ? q + 1 : q));
            if (f != PFW_NO_MATCH) atomicMin(p.peer_first[o] + off, f);
            if (p.peer_comps) atomicAdd(p.peer_comps[o] + off, c);
        } else {
            for (int t = 0; t < p.npeers; t++) {
                if (f != PFW_NO_MATCH) atomicMin(p.peer_first[t] + id, f);
                if (p.peer_comps) atomicAdd(p.peer_comps[t] + id, c);
            }
        }
    } else {
        const uint32_t fo = f != PFW_NO_MATCH ? f : p.nomatch_out;
        const uint8_t vo = (fl != PFW_NO_MATCH) ? p.accept[fl] : (uint8_t)0;
        if (CS) {
            // match-set scans write each packet's results once, in packet
            // order: streaming stores (evict-first in L2), so the output
            // stream does not push the tables out (the rule scan's scattered
            // per-pass writes keep the default policy: partial sectors)
            __stcs(p.first + id, fo);
            if (p.comps) __stcs(p.comps + id, c);
            if (p.verdict) __stcs(reinterpret_cast<signed char *>(p.verdict + id), (signed char)vo);
        } else {
            p.first[id] = fo;
            if (p.comps) p.comps[id] = c;
            if (p.verdict) p.verdict[id] = vo;
        }
    }
    st_sum += c;
    st_max = max(st_max, c);
}

__device__ __forceinline__ uint32_t sub_fma(uint32_t x, uint32_t one, uint32_t nlo) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(nlo));
    return d;
}

// Fast-path test.  FMA: IP subtractions as IMAD with a runtime 1 (FMA-heavy
// pipe) instead of IADD3 (ALU pipe, the bottleneck).
template <bool FMA, bool CH = false>
__device__ __forceinline__ bool rule_test(const uint32_t (&r)[NF], uint32_t src, uint32_t dst, float A,
                                          float A2, float B, uint32_t one) {
    uint32_t a, b;
    if (FMA) {
        a = sub_fma(src, one, r[F_SRC_NLO]);
        b = sub_fma(dst, one, r[F_DST_NLO]);
    } else {
        a = src + r[F_SRC_NLO];
        b = dst + r[F_DST_NLO];
    }
    // A holds D = A - A2 (packet precompute): dA = D*c1 + (A2 - loA) is
    // A - loA for c1 = 1 and A2 - loA for c1 = 0, exactly (integers < 2^24).
    // CH (protocol-split chain tables): every rule is encoded protocol-free
    // (c1 = 0), so dA = A2 - loA is one FADD.
    const float x = A2 + __uint_as_float(r[F_A_NLO]);
    const float dA = CH ? x : fmaf(A, __uint_as_float(r[F_A_C1]), x);
    const float dB = B + __uint_as_float(r[F_B_NLO]);
    return (a <= r[F_SRC_W]) & (b <= r[F_DST_W]) & (__float_as_uint(dA) <= r[F_A_W]) &
           (__float_as_uint(dB) <= r[F_B_W]);
}

// The two halves of the fast-path test, for warp-level short-circuit
// evaluation (SC): the IP prefix tests first (they pass for ~1% of random
// rule/packet pairs), the port/protocol tests only for rows where some lane
// passed them -- model.py:224-230 evaluates the conjunction lazily too.
template <bool FMA>
__device__ __forceinline__ bool ip_test(const uint32_t (&r)[NF], uint32_t src, uint32_t dst, uint32_t one) {
    uint32_t a, b;
    if (FMA) {
        a = sub_fma(src, one, r[F_SRC_NLO]);
        b = sub_fma(dst, one, r[F_DST_NLO]);
    } else {
        a = src + r[F_SRC_NLO];
        b = dst + r[F_DST_NLO];
    }
    return (a <= r[F_SRC_W]) & (b <= r[F_DST_W]);
}

__device__ __forceinline__ bool port_test(const uint32_t (&r)[NF], float A, float A2, float B) {
    const float x = A2 + __uint_as_float(r[F_A_NLO]);
    const float dA = fmaf(A, __uint_as_float(r[F_A_C1]), x);
    const float dB = B + __uint_as_float(r[F_B_NLO]);
    return (__float_as_uint(dA) <= r[F_A_W]) & (__float_as_uint(dB) <= r[F_B_W]);
}

// Slow-path re-evaluation (once per packet, after a stage hit).  Written with a
// different instruction sequence so the compiler cannot CSE it with the fast
// path and keep KS predicates / values alive across the vote.  Exact for the
// same reasons: all float operands are integers < 2^24 and c1, c2 are 0 or 1.
template <bool FMA, bool CH = false>
__device__ __forceinline__ bool rule_test_slow(const uint32_t (&r)[NF], uint32_t src, uint32_t dst,
                                               float A, float A2, float B, uint32_t one) {
    uint32_t a, b;
    if (FMA) {
        a = src + r[F_SRC_NLO];
        b = dst + r[F_DST_NLO];
    } else {
        a = sub_fma(src, one, r[F_SRC_NLO]);
        b = sub_fma(dst, one, r[F_DST_NLO]);
    }
    const float dA = CH ? __fsub_rn(A2, -__uint_as_float(r[F_A_NLO]))
                        : __fadd_rn(__fmul_rn(A, __uint_as_float(r[F_A_C1])),
                                    __fsub_rn(A2, -__uint_as_float(r[F_A_NLO])));
    const float dB = __fsub_rn(B, -__uint_as_float(r[F_B_NLO]));
    return (a <= r[F_SRC_W]) & (b <= r[F_DST_W]) & (__float_as_uint(dA) <= r[F_A_W]) &
           (__float_as_uint(dB) <= r[F_B_W]);
}

// Stage-local first match among rows [J0, J1) for one packet (some lane hit
// there): rows in rule order, one ballot each, stop at the first non-empty.
template <int KS, int J0, int J1, bool FMA, bool CH>
__device__ __forceinline__ unsigned rows_first(const uint32_t (&r)[KS][NF], uint32_t src, uint32_t dst,
                                               float A, float A2, float B, uint32_t one) {
#pragma unroll
    for (int j = J0; j < J1; j++) {
        const unsigned b = __ballot_sync(0xFFFFFFFFu, rule_test_slow<FMA, CH>(r[j], src, dst, A, A2, B, one));
        if (b) return (unsigned)(j * 32 + __ffs(b) - 1);
    }
    return 0xFFFFFFFFu;  // unreachable when the caller's vote hit
}

// Slow path: the stage hit; the half-stage accumulators say which half holds
// the first match, so at most KS/2 rows are re-evaluated.
template <int KS, bool FMA, bool CH>
__device__ __forceinline__ unsigned stage_first(const uint32_t (&r)[KS][NF], bool accA, uint32_t src,
                                                uint32_t dst, float A, float A2, float B, uint32_t one) {
    if (__any_sync(0xFFFFFFFFu, accA)) return rows_first<KS, 0, KS / 2, FMA, CH>(r, src, dst, A, A2, B, one);
    return rows_first<KS, KS / 2, KS, FMA, CH>(r, src, dst, A, A2, B, one);
}

// protocol of tile slot i from the shared-memory packet words (B = dport<<8 | proto)
__device__ __forceinline__ uint32_t s_pk_proto(const uint4 *, const uint32_t *s_pr, int i) {
    return ((uint32_t)__uint_as_float(s_pr[i])) & 0xFFu;
}

// One warp, P live packets of the tile (warp-uniform), one stage of KS rows in
// registers: the fast path ORs each packet's row results into two half-stage
// accumulators; a packet whose stage hit locates its first match with the
// slow path and records it.  P independent packets = P-fold ILP.
template <int P, int KS, bool FMA, bool HALF, bool CH>
__device__ __forceinline__ void scan_group(const uint32_t (&r)[KS][NF], const int (&q)[P],
                                           const uint4 *s_pk, const uint32_t *s_pr, uint32_t *s_first,
                                           int64_t s, uint32_t one, int lane) {
    uint4 v[P];
    float a[P], c[P], b[P];
#pragma unroll
    for (int k = 0; k < P; k++) {
        v[k] = s_pk[q[k]];
        b[k] = __uint_as_float(s_pr[q[k]]);
        a[k] = __uint_as_float(v[k].z);
        c[k] = __uint_as_float(v[k].w);
    }
    // HALF: two half-stage accumulators per packet (the slow path then
    // re-checks <= KS/2 rows); with HALF off one accumulator per packet keeps
    // the live predicates within the 7 predicate registers for larger P.
    bool lo[P], hi[P];
#pragma unroll
    for (int k = 0; k < P; k++) lo[k] = hi[k] = false;
#pragma unroll
    for (int j = 0; j < KS; j++)
#pragma unroll
        for (int k = 0; k < P; k++) {
            const bool m = rule_test<FMA, CH>(r[j], v[k].x, v[k].y, a[k], c[k], b[k], one);
            if (HALF && j >= KS / 2) hi[k] |= m; else lo[k] |= m;
        }
    // one vote for the whole group; per-packet votes only when it hit
    bool any = false;
#pragma unroll
    for (int k = 0; k < P; k++) any |= lo[k] | hi[k];
    if (!__any_sync(0xFFFFFFFFu, any)) return;
#pragma unroll
    for (int k = 0; k < P; k++) {
        if (__any_sync(0xFFFFFFFFu, lo[k] | hi[k])) {
            const unsigned f =
                HALF ? stage_first<KS, FMA, CH>(r, lo[k], v[k].x, v[k].y, a[k], c[k], b[k], one)
                     : rows_first<KS, 0, KS, FMA, CH>(r, v[k].x, v[k].y, a[k], c[k], b[k], one);
            PFW_CHECK(f < (unsigned)KS * 32u && q[k] >= 0);
            if (lane == 0) s_first[q[k]] = (uint32_t)(s + f);
        }
    }
}

#ifndef PFW_GROUP_HALF
#define PFW_GROUP_HALF 0
#endif
#ifndef PFW_GROUP
#define PFW_GROUP 3
#endif

// One stage over this warp's share of the live list: groups of GROUP packets
// (independent chains for ILP, loop overhead shared by the group).  CH: the
// sport/proto test is the one-FADD protocol-free/-fixed form.
template <int KS, bool FMA, bool CH>
__device__ __forceinline__ void scan_live(const uint32_t (&r)[KS][NF], const uint16_t *live, int nlive,
                                          int warp, const uint4 *s_pk, const uint32_t *s_pr,
                                          uint32_t *s_first, int64_t s, uint32_t one, int lane) {
    constexpr int NW = 8;  // warps per CTA (BLOCK / 32)
    constexpr int G = PFW_GROUP;
    int i = warp;
    for (; i + (G - 1) * NW < nlive; i += G * NW) {
        int qq[G];
#pragma unroll
        for (int k = 0; k < G; k++) qq[k] = live[i + k * NW];
        scan_group<G, KS, FMA, (PFW_GROUP_HALF != 0), CH>(r, qq, s_pk, s_pr, s_first, s, one, lane);
    }
    if (G > 3 && i + NW < nlive) {
        const int qq[2] = {live[i], live[i + NW]};
        scan_group<2, KS, FMA, true, CH>(r, qq, s_pk, s_pr, s_first, s, one, lane);
        i += 2 * NW;
    }
    if (i + NW < nlive) {
        const int qq[2] = {live[i], live[i + NW]};
        scan_group<2, KS, FMA, true, CH>(r, qq, s_pk, s_pr, s_first, s, one, lane);
        i += 2 * NW;
    }
    if (i < nlive) {
        const int qq[1] = {live[i]};
        scan_group<1, KS, FMA, true, CH>(r, qq, s_pk, s_pr, s_first, s, one, lane);
    }
}

constexpr int BLOCK = 256;
constexpr int NWARPS = BLOCK / 32;

// shared-memory layout for a tile of T packets (T <= 65535)
__host__ __device__ constexpr size_t smem_bytes(int T, int KS) {
    return (size_t)T * 16      // packet {src, dst, A, A2}
           + (size_t)T * 4     // packet B
           + (size_t)T * 4     // packet id
           + (size_t)T * 4     // first
           + (size_t)T * 2 * 2 // live lists (ping-pong)
           + 2 * (size_t)NF * 32 * KS * 4  // rule stage ring (2 buffers)
           + 64;               // mbarriers + counters
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void *sdst, const void *gsrc, unsigned bytes,
                                             uint64_t *bar) {
    unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
    unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(gsrc), "r"(bytes), "r"(b)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Issue the TMA copies of one stage (NF field rows of 32*KS words each).
// Stage start `s` is 32-aligned relative to the table (the kernel aligns lo
// down and masks the rules below lo), so every row copy is 16B aligned.
template <int KS>
__device__ __forceinline__ void issue_stage(const ScanParams &p, int64_t s, uint32_t *buf,
                                            uint64_t *bar) {
    constexpr unsigned ROW = 32 * KS * 4;
    mbar_expect_tx(bar, NF * ROW);
#pragma unroll
    for (int f = 0; f < NF; f++) tma_bulk_g2s(buf + f * 32 * KS, p.rules + f * p.rpad + s, ROW, bar);
}

// 8-row stages need ~120 registers (2 CTAs = 16 warps per SM); short stages
// fit 3 CTAs per SM (24 warps) for more latency hiding.
template <int KS>
constexpr int min_ctas() { return KS <= 4 ? 3 : 2; }

template <int KS, int MODE, bool FMA, bool SC, bool CH>
__global__ void __launch_bounds__(BLOCK, min_ctas<KS>()) scan_kernel(ScanParams p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int TMAX = p.tile;  // shared-memory capacity in packets
    uint4 *s_pk = reinterpret_cast<uint4 *>(smem_raw);
    uint32_t *s_rules = reinterpret_cast<uint32_t *>(s_pk + TMAX);      // 2 * NF * 32 * KS
    uint32_t *s_pr = s_rules + 2 * NF * 32 * KS;
    uint32_t *s_id = s_pr + TMAX;
    uint32_t *s_first = s_id + TMAX;
    uint16_t *s_liveA = reinterpret_cast<uint16_t *>(s_first + TMAX);
    uint16_t *s_liveB = s_liveA + TMAX;
    uint64_t *s_bar = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(s_liveB + TMAX) + 15) & ~uintptr_t(15));
    int *s_misc = reinterpret_cast<int *>(s_bar + 2);  // [0],[2] live counts, [1] tile, [3],[4] proto min/max

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t one = p.one;
    constexpr int STAGE = 32 * KS;
    const bool final_pass = p.out_ids == nullptr;
    int64_t count = p.in_count ? (int64_t)*p.in_count : p.n;
    const uint32_t *in_ids = p.in_ids ? p.in_ids + (p.bucket_base ? *p.bucket_base : 0u) : nullptr;
    if (p.bk_single && *p.bk_single >= 0) {
        // single-protocol batch: the bucket list was not written; the only
        // non-empty bucket is the whole batch in order
        in_ids = nullptr;
        count = (*p.bk_single == p.bk_index) ? p.n : 0;
    }
    // Tile size for this pass: the full capacity when there is enough work;
    // otherwise sized so the tile count is a whole number of waves of the
    // persistent grid (small batches and late passes carry few packets: a
    // 1.3-wave tail would idle most SMs).  Every CTA derives the same T.
    int T = TMAX;
    {
        const int64_t g = (int64_t)gridDim.x;
        const int64_t k = (count + g * TMAX - 1) / (g * TMAX);  // waves at the full tile size
        if (k >= 1) {
            const int64_t want = ((count + g * k - 1) / (g * k) + 31) & ~int64_t(31);
            if (want < T) T = (int)(want < 64 ? 64 : want);
        }
    }
    const int64_t ntiles = (count + T - 1) / T;

    unsigned long long st_sum = 0;
    unsigned st_max = 0;

    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned phase = 0u;  // bit b = parity of barrier b
    __syncthreads();

    for (;;) {
        if (tid == 0) s_misc[1] = (int)atomicAdd(p.tile_counter, 1u);
        __syncthreads();
        const int64_t tile = s_misc[1];
        if (tile >= ntiles) break;
        const int64_t base = tile * T;
        const int cnt = (int)((count - base) < T ? (count - base) : (int64_t)T);

        // prefetch the pass's first stage while the packet tile loads
        const bool any_rules = p.s_begin < p.s_end;
        if (tid == 0 && any_rules) {
            fence_proxy_async();
            issue_stage<KS>(p, p.s_begin, s_rules, &s_bar[0]);
        }

        for (int i = tid; i < cnt; i += BLOCK) {
            // per-packet precompute, amortised over every stage of the pass:
            // the fp32 port/proto words (exact integers < 2^24)
            const uint32_t id = in_ids ? __ldg(in_ids + base + i) : (uint32_t)(base + i);
            PFW_CHECK(id < (uint64_t)p.n && i < T && T <= TMAX);
            uint4 v;
            if (p.pkts) {
                v = __ldg(p.pkts + id);
            } else {
                v.x = __ldg(p.cols.src + id);
                v.y = __ldg(p.cols.dst + id);
                v.z = ((uint32_t)__ldg(p.cols.sport + id) << 16) | (uint32_t)__ldg(p.cols.dport + id);
                v.w = __ldg(p.cols.proto + id);
            }
            const uint32_t sp = v.z >> 16, dp = v.z & 0xFFFFu, pr = v.w & 0xFFu;
            const float fa = (float)((pr << 16) | sp), fa2 = (float)((sp << 8) | pr);
            s_pk[i] = make_uint4(v.x, v.y, __float_as_uint(fa - fa2), __float_as_uint(fa2));
            s_pr[i] = __float_as_uint((float)((dp << 8) | pr));
            s_id[i] = id;
            s_first[i] = PFW_NO_MATCH;
            s_liveA[i] = (uint16_t)i;
        }
        // is the tile protocol-uniform?  (warp min/max, one smem atomic per warp)
        if (!CH && !SC) {
            if (tid == 0) {
                s_misc[3] = 255;
                s_misc[4] = 0;
            }
            __syncthreads();
            unsigned pmin = 255u, pmax = 0u;
            for (int i = tid; i < cnt; i += BLOCK) {
                const uint32_t pr = s_pk_proto(s_pk, s_pr, i);
                pmin = min(pmin, pr);
                pmax = max(pmax, pr);
            }
            pmin = __reduce_min_sync(0xFFFFFFFFu, pmin);
            pmax = __reduce_max_sync(0xFFFFFFFFu, pmax);
            if (lane == 0) {
                atomicMin(&s_misc[3], (int)pmin);
                atomicMax(&s_misc[4], (int)pmax);
            }
        }
        __syncthreads();
        // (the short-circuit variant keeps the generic encoding)
        const bool tile_uniform = !CH && !SC && s_misc[3] == s_misc[4];
        const uint32_t tile_proto = (uint32_t)s_misc[3];
        if (tile_uniform) {
            // A2 slot <- the protocol-major word A = D + A2 (exact integers)
            for (int i = tid; i < cnt; i += BLOCK) {
                const uint4 v = s_pk[i];
                s_pk[i].w = __float_as_uint(__uint_as_float(v.z) + __uint_as_float(v.w));
            }
            __syncthreads();
        }

        int nlive = any_rules ? cnt : 0;
        uint16_t *live = s_liveA, *live2 = s_liveB;
        int buf = 0, kc = 0;
        int64_t s = p.s_begin;
        while (nlive > 0 && s < p.s_end) {
            // prefetch next stage into the other buffer (its previous reader
            // finished: every warp passed the __syncthreads that ended it)
            const int64_t sn = s + STAGE;
            if (tid == 0 && sn < p.s_end) {
                fence_proxy_async();
                issue_stage<KS>(p, sn, s_rules + (buf ^ 1) * NF * STAGE, &s_bar[buf ^ 1]);
            }
            mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;

            // stage rules -> registers (lane l: rules s + 32j + l)
            const uint32_t *sr = s_rules + buf * NF * STAGE;
            PFW_CHECK(s >= 0 && s + STAGE <= p.rpad && nlive <= T);
            uint32_t r[KS][NF];
#pragma unroll
            for (int j = 0; j < KS; j++) {
#pragma unroll
                for (int f = 0; f < NF; f++) r[j][f] = sr[f * STAGE + j * 32 + lane];
                const int64_t ri = s + j * 32 + lane;
                if (ri < p.lo || ri >= p.hi) {
                    r[j][F_B_NLO] = NEVER_B_NLO;
                    r[j][F_B_W] = NEVER_B_W;
                }
            }
            // Live packets are split across the warps (warp-uniform, so every
            // branch below is warp-uniform too).
            int i = warp;
            if (!SC) {
                if (CH || !tile_uniform) {
                    scan_live<KS, FMA, CH>(r, live, nlive, warp, s_pk, s_pr, s_first, s, one, lane);
                } else {
                    // every packet of the tile has protocol tile_proto: rewrite the
                    // ANY rules' sport test into the protocol-major form for that
                    // protocol (concrete rules already have it), so every rule --
                    // still tested against every packet -- needs one FADD
#pragma unroll
                    for (int j = 0; j < KS; j++) {
                        if (r[j][F_A_C1] == 0u) {  // c1 = +0.0f: ANY rule, A2 encoding
                            const uint32_t slo = ((uint32_t)(-__uint_as_float(r[j][F_A_NLO]))) >> 8;
                            const uint32_t shi = (((uint32_t)__uint_as_float(r[j][F_A_W])) + (slo << 8)) >> 8;
                            r[j][F_A_NLO] = __float_as_uint(-(float)((tile_proto << 16) | slo));
                            r[j][F_A_W] = __float_as_uint((float)(shi - slo));
                        }
                    }
                    scan_live<KS, FMA, true>(r, live, nlive, warp, s_pk, s_pr, s_first, s, one, lane);
                }
            } else {
                // short-circuit variant (off by default): rows in rule order; per
                // row the IP tests, one vote, the port/protocol tests only if some
                // lane passed them, and the ballot of the full result is the
                // exact first match (no stage-level OR, no re-evaluation)
                for (; i < nlive; i += NWARPS) {
                    const int q = live[i];
                    const uint4 v = s_pk[q];
                    const float bb = __uint_as_float(s_pr[q]);
                    const float a = __uint_as_float(v.z), c = __uint_as_float(v.w);
#pragma unroll
                    for (int j = 0; j < KS; j++) {
                        const bool ip = ip_test<FMA>(r[j], v.x, v.y, one);
                        if (__any_sync(0xFFFFFFFFu, ip)) {
                            const unsigned bm = __ballot_sync(0xFFFFFFFFu, ip & port_test(r[j], a, c, bb));
                            if (bm) {
                                if (lane == 0) s_first[q] = (uint32_t)(s + j * 32 + __ffs(bm) - 1);
                                break;
                            }
                        }
                    }
                }
            }
            // live counter alternates between two slots so that resetting one
            // never races with a late reader of the previous stage's count
            int *ctr = &s_misc[kc ? 2 : 0];
            if (tid == 0) *ctr = 0;
            __syncthreads();
            // retire matched packets: compact the live list (order is free)
            for (int i0 = 0; i0 < nlive; i0 += BLOCK) {
                const int i = i0 + tid;
                int q = 0;
                bool keep = false;
                if (i < nlive) {
                    q = live[i];
                    keep = s_first[q] == PFW_NO_MATCH;
                }
                const unsigned b = __ballot_sync(0xFFFFFFFFu, keep);
                int off = 0;
                if (lane == 0 && b) off = atomicAdd(ctr, __popc(b));
                off = __shfl_sync(0xFFFFFFFFu, off, 0);
                if (keep) live2[off + __popc(b & ((1u << lane) - 1u))] = (uint16_t)q;
            }
            __syncthreads();
            nlive = *ctr;
            kc ^= 1;
            uint16_t *t = live;
            live = live2;
            live2 = t;
            buf ^= 1;
            s = sn;
        }
        // drain a prefetched stage that was not consumed (tile ended early)
        if (any_rules && s < p.s_end) {
            mbar_wait(&s_bar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
        }

        // epilogue: resolve matched packets (and, in the final pass, the
        // unmatched ones); survivors of a non-final pass go to the next pass
        const uint32_t span = (uint32_t)(p.win_hi > p.win_lo ? p.win_hi - p.win_lo : 0);
        for (int i0 = 0; i0 < cnt; i0 += BLOCK) {
            const int i = i0 + tid;
            bool survive = false;
            uint32_t id = 0;
            if (i < cnt) {
                uint32_t f = s_first[i];
                id = s_id[i];
                survive = !final_pass && f == PFW_NO_MATCH;
                if (!survive) {
                    PFW_CHECK(f == PFW_NO_MATCH || (f >= p.lo && f < p.hi));
                    if (p.orig && f != PFW_NO_MATCH) f = __ldg(p.orig + f);
                    PFW_CHECK(f == PFW_NO_MATCH || (f >= p.win_lo && f < p.win_hi));
                    emit_result<MODE>(p, id, f, span, st_sum, st_max);
                }
            }
            const unsigned b = __ballot_sync(0xFFFFFFFFu, survive);
            if (b) {
                unsigned off = 0;
                if (lane == 0) off = atomicAdd(p.out_count, (unsigned)__popc(b));
                off = __shfl_sync(0xFFFFFFFFu, off, 0);
                if (survive) {
                    PFW_CHECK(off + __popc(b & ((1u << lane) - 1u)) < (uint64_t)p.out_cap);
                    p.out_ids[off + __popc(b & ((1u << lane) - 1u))] = id;
                }
            }
        }
        __syncthreads();
    }
    if (p.stats) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            st_sum += __shfl_xor_sync(0xFFFFFFFFu, st_sum, o);
            st_max = max(st_max, __shfl_xor_sync(0xFFFFFFFFu, st_max, o));
        }
        if (lane == 0) {
            if (st_sum) atomicAdd(&p.stats[0], st_sum);
            if (st_max) atomicMax(&p.stats[1], (unsigned long long)st_max);
        }
    }
}

// ---------------------------------------------------- protocol bucketing
// Packets grouped by rule chain (protocol): per-block shared-memory histograms
// and one global atomic per chain per block, so single-protocol traffic does
// not serialise on one counter.  counts/base/cursor live in bc[0..3*MAX_CHAINS).
constexpr int BK_BLOCK = 256, BK_PER_THREAD = 16;

__device__ __forceinline__ uint32_t pkt_proto(const uint4 *pkts, const uint8_t *proto_col, int64_t i) {
    return proto_col ? (uint32_t)__ldg(proto_col + i) : __ldg(&pkts[i].w) & 0xFFu;
}

__global__ void __launch_bounds__(BK_BLOCK) bucket_count_kernel(const uint4 *pkts, const uint8_t *proto_col,
                                                                int64_t n, const uint8_t *lut, int nchains,
                                                                unsigned *bc) {
    __shared__ unsigned hist[MAX_CHAINS];
    for (int c = threadIdx.x; c < nchains; c += BK_BLOCK) hist[c] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * BK_BLOCK * BK_PER_THREAD;
    for (int k = 0; k < BK_PER_THREAD; k++) {
        const int64_t i = b0 + (int64_t)k * BK_BLOCK + threadIdx.x;
        if (i < n) atomicAdd(&hist[lut[pkt_proto(pkts, proto_col, i)]], 1u);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nchains; c += BK_BLOCK)
        if (hist[c]) atomicAdd(&bc[c], hist[c]);
}

__global__ void bucket_prefix_kernel(int nchains, unsigned *bc, int *single) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned acc = 0;
        int nonempty = 0, last = -1;
        for (int c = 0; c < nchains; c++) {
            bc[MAX_CHAINS + c] = acc;  // base
            bc[2 * MAX_CHAINS + c] = 0;  // cursor
            acc += bc[c];
            if (bc[c]) {
                nonempty++;
                last = c;
            }
        }
        if (single) *single = nonempty == 1 ? last : -1;
    }
}

__global__ void __launch_bounds__(BK_BLOCK) bucket_scatter_kernel(const uint4 *pkts, const uint8_t *proto_col,
                                                                  int64_t n, const uint8_t *lut, int nchains,
                                                                  unsigned *bc, uint32_t *ids,
                                                                  const int *single) {
    if (single && *single >= 0) return;  // one bucket: scans read the batch in order
    __shared__ unsigned hist[MAX_CHAINS], gbase[MAX_CHAINS];
    for (int c = threadIdx.x; c < nchains; c += BK_BLOCK) hist[c] = 0;
    __syncthreads();
    const int64_t b0 = (int64_t)blockIdx.x * BK_BLOCK * BK_PER_THREAD;
    uint8_t ch[BK_PER_THREAD];
#pragma unroll
    for (int k = 0; k < BK_PER_THREAD; k++) {
        const int64_t i = b0 + (int64_t)k * BK_BLOCK + threadIdx.x;
        ch[k] = i < n ? lut[pkt_proto(pkts, proto_col, i)] : 0;
        if (i < n) atomicAdd(&hist[ch[k]], 1u);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nchains; c += BK_BLOCK) {
        gbase[c] = hist[c] ? bc[MAX_CHAINS + c] + atomicAdd(&bc[2 * MAX_CHAINS + c], hist[c]) : 0;
        hist[c] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK_PER_THREAD; k++) {
        const int64_t i = b0 + (int64_t)k * BK_BLOCK + threadIdx.x;
        if (i < n) {
            const unsigned pos = gbase[ch[k]] + atomicAdd(&hist[ch[k]], 1u);
            PFW_CHECK(pos < (uint64_t)n && ch[k] < nchains);
            ids[pos] = (uint32_t)i;
        }
    }
}

__global__ void acc_init_kernel(int64_t n, uint32_t *first, uint32_t *comps) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        first[i] = PFW_NO_MATCH;
        if (comps) comps[i] = 0;
    }
}

// e2e chunk of the function-parallel / hybrid models: verdicts from the
// combined first match, and the host's no-match value
__global__ void e2e_finish_kernel(const uint8_t *accept, uint32_t *first, uint8_t *verdict, int64_t n,
                                  uint32_t nomatch_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = first[i];
        if (verdict) verdict[i] = f != PFW_NO_MATCH ? accept[f] : (uint8_t)0;
        if (f == PFW_NO_MATCH) first[i] = nomatch_out;
    }
}

__global__ void verdict_kernel(const uint8_t *accept, const uint32_t *first, int64_t n,
                               uint8_t *verdict) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t f = first[i];
        verdict[i] = f != PFW_NO_MATCH ? accept[f] : 0;
    }
}

__global__ void combine_min_kernel(const uint32_t *rows, int64_t nrows, int64_t n, uint32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t m = PFW_NO_MATCH;
        for (int64_t w = 0; w < nrows; w++) m = min(m, rows[w * n + i]);
        out[i] = m;
    }
}

// ============================================================ generator
// xorshift64* is GF(2)-linear in its state, so the state after k steps is
// M^k s.  Matrices are stored as 64 columns: col[i] = M e_i.
struct Mat64 {
    uint64_t c[64];
};

__host__ __device__ inline uint64_t matvec(const uint64_t *col, uint64_t s) {
    uint64_t r = 0;
#pragma unroll 8
    for (int i = 0; i < 64; i++)
        if ((s >> i) & 1) r ^= col[i];
    return r;
}

inline uint64_t xs_step_state(uint64_t x) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
}

Mat64 mat_step() {
    Mat64 m;
    for (int i = 0; i < 64; i++) m.c[i] = xs_step_state(1ULL << i);
    return m;
}
Mat64 mat_mul(const Mat64 &a, const Mat64 &b) {  // a*b
    Mat64 r;
    for (int i = 0; i < 64; i++) r.c[i] = matvec(a.c, b.c[i]);
    return r;
}
Mat64 mat_pow(Mat64 m, uint64_t k) {
    Mat64 r;
    for (int i = 0; i < 64; i++) r.c[i] = 1ULL << i;
    while (k) {
        if (k & 1) r = mat_mul(r, m);
        m = mat_mul(m, m);
        k >>= 1;
    }
    return r;
}

constexpr int GEN_BLOCK = 128;
constexpr int GEN_PER_THREAD = 16;
constexpr int GEN_PER_BLOCK = GEN_BLOCK * GEN_PER_THREAD;  // packets per block
constexpr int GEN_LOG_BLOCK = 7;
__constant__ uint64_t c_jump[GEN_LOG_BLOCK][64];  // (M^(4*GEN_PER_THREAD))^(2^b)

struct GenParams {
    uint32_t proto, src_base, dst_base;
    uint64_t sspan, dspan;  // powers of two <= 2^32
    uint32_t sp_lo, dp_lo;
    uint64_t sp_n, dp_n;    // port counts (1..65536)
    uint64_t sp_lim, dp_lim;  // rejection limits (0 = power of two, never rejects)
};

__device__ __forceinline__ uint64_t xs_next(uint64_t &x) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x * 0x2545F4914F6CDD1DULL;
}

__global__ void __launch_bounds__(GEN_BLOCK) gen_kernel(GenParams g, const uint64_t *block_state,
                                                        int64_t start, int64_t n, uint4 *out,
                                                        unsigned long long *reject_at) {
    __shared__ uint4 stage[GEN_PER_BLOCK];
    const int64_t b0 = start + (int64_t)blockIdx.x * GEN_PER_BLOCK;
    uint64_t x = block_state[blockIdx.x];
    for (int bit = 0; bit < GEN_LOG_BLOCK; bit++)
        if ((threadIdx.x >> bit) & 1) x = matvec(c_jump[bit], x);
    const int64_t p0 = b0 + (int64_t)threadIdx.x * GEN_PER_THREAD;
    bool rej = false;
    int64_t rej_at = 0;
    for (int k = 0; k < GEN_PER_THREAD; k++) {
        const uint64_t d0 = xs_next(x), d1 = xs_next(x), d2 = xs_next(x), d3 = xs_next(x);
        if (!rej && ((g.sp_lim && d1 >= g.sp_lim) || (g.dp_lim && d3 >= g.dp_lim))) {
            rej = true;
            rej_at = p0 + k;
        }
        uint4 v;
        v.x = g.src_base + (uint32_t)(d0 & (g.sspan - 1));
        const uint32_t sp = g.sp_lo + (uint32_t)(d1 % g.sp_n);
        v.y = g.dst_base + (uint32_t)(d2 & (g.dspan - 1));
        const uint32_t dp = g.dp_lo + (uint32_t)(d3 % g.dp_n);
        v.z = (sp << 16) | dp;
        v.w = g.proto;
        stage[threadIdx.x * GEN_PER_THREAD + k] = v;
    }
    if (rej && rej_at < n) atomicMin(reject_at, (unsigned long long)rej_at);
    __syncthreads();
    for (int i = threadIdx.x; i < GEN_PER_BLOCK; i += GEN_BLOCK) {
        const int64_t q = b0 + i;
        if (q < n) out[q] = stage[i];
    }
}

uint64_t host_seed_state(uint64_t seed) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z ? z : 0x9E3779B97F4A7C15ULL;
}

uint64_t host_next(uint64_t &x) {
    x = xs_step_state(x);
    return x * 0x2545F4914F6CDD1DULL;
}

uint64_t host_randbelow(uint64_t &x, uint64_t n) {
    const uint64_t rem = (0 - n) % n;
    if (rem == 0) return host_next(x) % n;
    const uint64_t lim = 0 - rem;
    for (;;) {
        const uint64_t r = host_next(x);
        if (r < lim) return r % n;
    }
}


#include "matchset.cuh"

int ensure_ws(ScanWs &ws, int64_t n) {
    if (!ws.ctr) CUDA_TRY(cudaMalloc(&ws.ctr, 2 * MAX_PASSES * sizeof(unsigned int)));
    if (ws.cap < n) {
        if (ws.ids) cudaFree(ws.ids);
        ws.ids = nullptr;
        ws.cap = 0;
        const int64_t cap = n < 4096 ? 4096 : n;
        CUDA_TRY(cudaMalloc(&ws.ids, 2 * (size_t)cap * sizeof(uint32_t)));
        ws.cap = cap;
    }
    return PFW_OK;
}

void free_ws(ScanWs &ws) {
    if (ws.ids) cudaFree(ws.ids);
    if (ws.ctr) cudaFree(ws.ctr);
    if (ws.d_bucket) cudaFree(ws.d_bucket);
    if (ws.d_bcount) cudaFree(ws.d_bcount);
    ws = ScanWs{};
}

// Pass plan over the window [lo, hi): stage-aligned boundaries starting at
// lo & ~31, first pass g_first_pass rules, then doubling.  Each pass scans
// only the packets the previous passes left unmatched, compacted into dense
// tiles, so the long tail of late-matching / default-deny packets never runs
// on near-empty tiles.
std::vector<int64_t> plan_passes(int64_t lo, int64_t hi, int stage) {
    std::vector<int64_t> b;
    const int64_t s0 = lo & ~int64_t(31);
    b.push_back(s0);
    if (lo >= hi) {
        b.push_back(s0);
        return b;
    }
    int64_t len = g_first_pass > 0 ? ((g_first_pass + stage - 1) / stage) * (int64_t)stage : 0;
    int64_t cur = s0;
    while (len > 0 && cur + len < hi && (int)b.size() < MAX_PASSES) {
        cur += len;
        b.push_back(cur);
        len *= 2;
    }
    b.push_back(hi);
    return b;
}

template <int KS, int MODE, bool FMA, bool SC, bool CH = false>
int launch_scan_t(pfw_ruleset *h, const ScanParams &p0, ScanWs &ws, cudaStream_t st) {
    const size_t sm = smem_bytes(p0.tile, KS);
    auto kern = scan_kernel<KS, MODE, FMA, SC, CH>;
    int maxsm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    if (sm > (size_t)maxsm)
        return set_err(PFW_ERR_INVALID, "tile %d x ks %d needs %zu B of shared memory (max %d)", p0.tile,
                       KS, sm, maxsm);
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int occ = g_ctas_per_sm;
    if (occ <= 0) {
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, BLOCK, sm));
        if (occ < 1) occ = 1;
    }
    const int64_t ntiles0 = (p0.n + 255) / 256;  // smallest tile the kernel adapts to
    int64_t grid = (int64_t)h->sms * occ;
    if (grid > ntiles0) grid = ntiles0;
    if (grid < 1) grid = 1;

    const std::vector<int64_t> b = plan_passes(p0.lo, p0.hi, 32 * KS);
    const int npass = (int)b.size() - 1;
    if (npass > 1) {
        int rc = ensure_ws(ws, p0.n);
        if (rc != PFW_OK) return rc;
    } else if (!ws.ctr) {
        CUDA_TRY(cudaMalloc(&ws.ctr, 2 * MAX_PASSES * sizeof(unsigned int)));
    }
    CUDA_TRY(cudaMemsetAsync(ws.ctr, 0, 2 * (size_t)npass * sizeof(unsigned int), st));
    for (int k = 0; k < npass; k++) {
        ScanParams p = p0;
        p.s_begin = b[k];
        p.s_end = b[k + 1];
        p.tile_counter = ws.ctr + 2 * k;
        p.in_ids = k == 0 ? p0.in_ids0 : ws.ids + (size_t)((k - 1) & 1) * ws.cap;
        p.in_count = k == 0 ? p0.in_count0 : ws.ctr + 2 * (k - 1) + 1;
        p.bucket_base = k == 0 ? p0.bucket_base : nullptr;
        p.bk_single = k == 0 ? p0.bk_single : nullptr;
        const bool last = k == npass - 1;
        p.out_ids = last ? nullptr : ws.ids + (size_t)(k & 1) * ws.cap;
        p.out_count = last ? nullptr : ws.ctr + 2 * k + 1;
        p.out_cap = last ? 0 : ws.cap;
        kern<<<(unsigned)grid, BLOCK, sm, st>>>(p);
        CUDA_TRY(cudaGetLastError());
        g_launches++;
    }
    return PFW_OK;
}

template <int MODE, bool FMA, bool SC>
int launch_scan_ks(pfw_ruleset *h, const ScanParams &p, ScanWs &ws, cudaStream_t st) {
    // protocol-split chain tables: the protocol-free variant (default KS / FMA / no SC)
    if (p.chain && g_ks == 8 && FMA && !SC) return launch_scan_t<8, MODE, true, false, true>(h, p, ws, st);
    switch (g_ks) {
        case 2: return launch_scan_t<2, MODE, FMA, SC>(h, p, ws, st);
        case 4: return launch_scan_t<4, MODE, FMA, SC>(h, p, ws, st);
        case 6: return launch_scan_t<6, MODE, FMA, SC>(h, p, ws, st);
        case 8: return launch_scan_t<8, MODE, FMA, SC>(h, p, ws, st);
        default: return set_err(PFW_ERR_INVALID, "unsupported ks=%d (2, 4, 6 or 8)", g_ks);
    }
}

template <int MODE, bool SC>
int launch_scan_fma(pfw_ruleset *h, const ScanParams &p, ScanWs &ws, cudaStream_t st) {
    return g_force_imad ? launch_scan_ks<MODE, true, SC>(h, p, ws, st)
                        : launch_scan_ks<MODE, false, SC>(h, p, ws, st);
}

template <int MODE>
int launch_scan_sc(pfw_ruleset *h, const ScanParams &p, ScanWs &ws, cudaStream_t st) {
    return g_short_circuit ? launch_scan_fma<MODE, true>(h, p, ws, st)
                           : launch_scan_fma<MODE, false>(h, p, ws, st);
}

int launch_mode(pfw_ruleset *h, int mode, const ScanParams &p, ScanWs &w, cudaStream_t st);
int launch_split(pfw_ruleset *h, int mode, const ScanParams &p, ScanWs &w, cudaStream_t st, bool chains);

int launch_scan(pfw_ruleset *h, int mode, int64_t lo, int64_t hi, const void *d_pkts, int64_t n,
                uint32_t *first, uint32_t *comps, uint8_t *verdict, uint64_t *stats,
                cudaStream_t st, ScanWs *ws = nullptr, const ScanParams *peer = nullptr,
                const PacketCols *cols = nullptr, uint32_t nomatch_out = PFW_NO_MATCH) {
    const bool acc = mode == MODE_ACC;
    if (!h) return set_err(PFW_ERR_INVALID, "null ruleset handle");
    if (n < 0) return set_err(PFW_ERR_INVALID, "negative packet count %lld", (long long)n);
    if (n > 0xFFFFFFFFll) return set_err(PFW_ERR_INVALID, "more than 2^32-1 packets in one call");
    if (lo < 0 || hi < 0) return set_err(PFW_ERR_INVALID, "negative rule window [%lld, %lld)",
                                         (long long)lo, (long long)hi);
    if (hi > h->n) return set_err(PFW_ERR_INVALID, "rule window end %lld beyond ruleset of %lld",
                                  (long long)hi, (long long)h->n);
    if (n == 0) return PFW_OK;
    NvtxRange nv(mode == MODE_ACC ? "pfw scan (accumulate)" : mode == MODE_PEER ? "pfw scan (fused peer combine)"
                                                                                : "pfw scan");
    const bool have_cols = cols && cols->proto && cols->src && cols->sport && cols->dst && cols->dport;
    if ((!d_pkts && !have_cols) || (!first && mode != MODE_PEER))
        return set_err(PFW_ERR_INVALID, "null packet or output pointer");
    if (acc && !comps) return set_err(PFW_ERR_INVALID, "accumulate needs a comps buffer");
    if (lo > hi) lo = hi;  // empty window: scan_range returns all -1
    ScanParams p{};
    p.rules = h->d_rules;
    p.accept = h->d_accept;
    p.rpad = h->rpad;
    p.lo = lo;
    p.hi = hi;
    p.win_lo = lo;
    p.win_hi = hi;
    p.orig = nullptr;
    p.pkts = have_cols ? nullptr : reinterpret_cast<const uint4 *>(d_pkts);
    if (have_cols) p.cols = *cols;
    p.n = n;
    p.first = first;
    p.comps = comps;
    p.verdict = verdict;
    p.stats = reinterpret_cast<unsigned long long *>(stats);
    p.tile = g_tile;
    p.one = 1;
    p.nomatch_out = nomatch_out;
    p.index_base = (uint32_t)h->index_base;
    DeviceGuard g(h->device);
    if (!g.ok) return set_err(PFW_ERR_CUDA, "cudaSetDevice(%d) failed", h->device);
    if (peer) {
        p.peer_first = peer->peer_first;
        p.peer_comps = peer->peer_comps;
        p.npeers = peer->npeers;
        p.scatter = peer->scatter;
    }
    ScanWs &w = ws ? *ws : h->ws;
    // match sets (matchset.cuh) unless the rule-by-rule scan is asked for
    // (algo 1, or one of its own options: protocol-split chains, short circuit)
    if (g_algo == 2 && !h->ms) return set_err(PFW_ERR_INVALID, "algo=2: this ruleset has no match sets");
    if (h->ms && (g_algo == 2 || (g_algo == 0 && !g_proto_split && !g_short_circuit)))
        return launch_ms(h, mode, p, st);
    if (g_proto_split && !h->chains.empty() && lo < hi) return launch_split(h, mode, p, w, st, true);
    // large batches are grouped by protocol first so that tiles are
    // protocol-uniform (the one-FADD sport test); single-protocol batches skip
    // the scatter on the device
    if (g_bucket && !h->chains.empty() && lo < hi && n >= g_bucket_min && !g_short_circuit)
        return launch_split(h, mode, p, w, st, false);
    return launch_mode(h, mode, p, w, st);
}

int launch_mode(pfw_ruleset *h, int mode, const ScanParams &p, ScanWs &w, cudaStream_t st) {
    switch (mode) {
        case MODE_ACC: return launch_scan_sc<MODE_ACC>(h, p, w, st);
        case MODE_PEER: return launch_scan_sc<MODE_PEER>(h, p, w, st);
        default: return launch_scan_sc<MODE_WRITE>(h, p, w, st);
    }
}

// Protocol-split scan: group the packets by rule chain on the device, then
// run the multi-pass scan of each chain over its bucket (empty buckets exit
// immediately; counts stay on the device, no host sync).
int launch_split(pfw_ruleset *h, int mode, const ScanParams &p0, ScanWs &w, cudaStream_t st,
                 bool chains) {
    const int nch = (int)h->chains.size();
    const int64_t n = p0.n;
    if (w.bucket_cap < n) {
        if (w.d_bucket) cudaFree(w.d_bucket);
        w.d_bucket = nullptr;
        w.bucket_cap = 0;
        CUDA_TRY(cudaMalloc(&w.d_bucket, (size_t)n * sizeof(uint32_t)));
        w.bucket_cap = n;
    }
    if (!w.d_bcount) CUDA_TRY(cudaMalloc(&w.d_bcount, (3 * MAX_CHAINS + 1) * sizeof(unsigned)));
    int *d_single = reinterpret_cast<int *>(w.d_bcount + 3 * MAX_CHAINS);
    CUDA_TRY(cudaMemsetAsync(w.d_bcount, 0, MAX_CHAINS * sizeof(unsigned), st));
    const unsigned nb = (unsigned)((n + BK_BLOCK * BK_PER_THREAD - 1) / (BK_BLOCK * BK_PER_THREAD));
    bucket_count_kernel<<<nb, BK_BLOCK, 0, st>>>(p0.pkts, p0.cols.proto, n, h->d_lut, nch, w.d_bcount);
    bucket_prefix_kernel<<<1, 32, 0, st>>>(nch, w.d_bcount, d_single);
    bucket_scatter_kernel<<<nb, BK_BLOCK, 0, st>>>(p0.pkts, p0.cols.proto, n, h->d_lut, nch, w.d_bcount,
                                                  w.d_bucket, d_single);
    CUDA_TRY(cudaGetLastError());
    g_launches += 3;
    // bucket c's ids start at base[c]; its count is bc[c].  The base is only
    // known on the device, so each chain scan reads its ids through a
    // device-side pointer computed by a tiny kernel into the ws pointer slot.
    for (int c = 0; c < nch; c++) {
        ScanParams p = p0;
        p.bucket_base = w.d_bcount + MAX_CHAINS + c;
        p.in_ids0 = w.d_bucket;
        p.in_count0 = w.d_bcount + c;
        p.bk_single = d_single;
        p.bk_index = c;
        if (chains) {  // protocol-split: this bucket scans its chain table
            const pfw_ruleset::Chain &ch = h->chains[(size_t)c];
            p.rules = ch.d_rules;
            p.rpad = ch.rpad;
            p.orig = ch.d_orig;
            p.chain = 1;
            p.win_lo = p0.lo;
            p.win_hi = p0.hi;
            p.lo = (int64_t)(std::lower_bound(ch.orig.begin(), ch.orig.end(), (uint32_t)p0.lo) - ch.orig.begin());
            p.hi = (int64_t)(std::lower_bound(ch.orig.begin(), ch.orig.end(), (uint32_t)p0.hi) - ch.orig.begin());
            if (p.lo >= p.hi) p.lo = p.hi;
        }  // else: protocol bucketing only -- the full table, protocol-uniform tiles
        int rc = launch_mode(h, mode, p, w, st);
        if (rc != PFW_OK) return rc;
    }
    return PFW_OK;
}

int grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 8) g = 148 * 8;
    return (int)(g < 1 ? 1 : g);
}


// L2 read-bandwidth probe for the match-set scan's access pattern (bench.py's
// roofline peak, measured on the same device in the same run): groups of 8
// lanes each read one random 128-byte line (16 bytes per lane) of an
// L2-resident buffer, K independent lines per lane in flight per iteration.
template <int K>
__global__ void __launch_bounds__(256) probe_l2_lines_kernel(const uint4 *__restrict__ p, uint32_t nlines,
                                                             int iters, uint32_t *sink) {
    const int lane = threadIdx.x & 31, grp = lane / 8, gl = lane % 8;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * 32u + (threadIdx.x >> 5) * 4u + (uint32_t)grp + 1u);
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint4 v[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            x = x * 1664525u + 1013904223u;  // group-uniform LCG
            const uint32_t line = (uint32_t)(((uint64_t)(x >> 8) * nlines) >> 24);
            v[k] = __ldg(p + (size_t)line * 8 + gl);
        }
#pragma unroll
        for (int k = 0; k < K; k++) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    if (acc == 0x12345678u) *sink = acc;  // keeps the loads
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

const char *pfw_last_error(void) { return g_err.c_str(); }

const char *pfw_version(void) {
    return "pfw " PFW_VERSION " sm_100a: match-set scan (per-field interval bitmaps, lane-group ballot) + "
           "rule-by-rule range-test grid (KS=2/4/6/8, TMA bulk stage ring)";
}

int pfw_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int pfw_probe_l2_lines(const void *d_buf, int64_t bytes, int lines_in_flight, int blocks_per_sm, int iters,
                       void *stream) {
    if (!d_buf || bytes < (1 << 20) || iters < 1 || blocks_per_sm < 1 || blocks_per_sm > 8)
        return set_err(PFW_ERR_INVALID, "bad probe arguments");
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    static uint32_t *sinks[64] = {};  // per device (the kernel's never-taken store target)
    if (dev < 0 || dev >= 64) return set_err(PFW_ERR_INVALID, "device %d out of range", dev);
    if (!sinks[dev]) CUDA_TRY(cudaMalloc(&sinks[dev], sizeof(uint32_t)));
    uint32_t *sink = sinks[dev];
    const uint32_t nlines = (uint32_t)std::min<int64_t>(bytes / 128, 0x7FFFFFFF);
    const auto *p = reinterpret_cast<const uint4 *>(d_buf);
    const cudaStream_t st = (cudaStream_t)stream;
    const unsigned grid = (unsigned)(sms * blocks_per_sm);
    switch (lines_in_flight) {
        case 2: probe_l2_lines_kernel<2><<<grid, 256, 0, st>>>(p, nlines, iters, sink); break;
        case 4: probe_l2_lines_kernel<4><<<grid, 256, 0, st>>>(p, nlines, iters, sink); break;
        case 8: probe_l2_lines_kernel<8><<<grid, 256, 0, st>>>(p, nlines, iters, sink); break;
        case 16: probe_l2_lines_kernel<16><<<grid, 256, 0, st>>>(p, nlines, iters, sink); break;
        default: return set_err(PFW_ERR_INVALID, "lines_in_flight: 2, 4, 8 or 16");
    }
    CUDA_TRY(cudaGetLastError());
    return PFW_OK;
}

int64_t pfw_launch_count(void) { return g_launches.load(); }

int pfw_read_counter(const char *name, int64_t *value) {
    if (!name || !value) return set_err(PFW_ERR_INVALID, "null argument");
    if (strcmp(name, "blocks_read")) return set_err(PFW_ERR_INVALID, "unknown counter '%s'", name);
    *value = 0;
    if (!g_counter_dev) return PFW_OK;
    unsigned long long v = 0;
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(&v, g_counter_dev, sizeof v, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemset(g_counter_dev, 0, sizeof v));
    *value = (int64_t)v;
    return PFW_OK;
}

static uint32_t f2u(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

int pfw_set_tuning(const char *key, int64_t value) {
    if (!key) return set_err(PFW_ERR_INVALID, "null key");
    if (!strcmp(key, "ks")) {
        if (value != 2 && value != 4 && value != 6 && value != 8)
            return set_err(PFW_ERR_INVALID, "ks must be 2, 4, 6 or 8");
        g_ks = (int)value;
    } else if (!strcmp(key, "tile")) {
        if (value < 256 || value > 8192 || value % 256) return set_err(PFW_ERR_INVALID, "tile must be a multiple of 256 in [256, 8192]");
        g_tile = (int)value;
    } else if (!strcmp(key, "ctas_per_sm")) {
        if (value < 0 || value > 8) return set_err(PFW_ERR_INVALID, "ctas_per_sm in [0, 8]");
        g_ctas_per_sm = (int)value;
    } else if (!strcmp(key, "first_pass")) {
        if (value < 0 || value > (1 << 24)) return set_err(PFW_ERR_INVALID, "first_pass in [0, 2^24]");
        g_first_pass = (int)value;
    } else if (!strcmp(key, "short_circuit")) {
        g_short_circuit = value != 0;
    } else if (!strcmp(key, "bucket")) {
        g_bucket = value != 0;
    } else if (!strcmp(key, "bucket_min")) {
        if (value < 0) return set_err(PFW_ERR_INVALID, "bucket_min must be >= 0");
        g_bucket_min = value;
    } else if (!strcmp(key, "proto_split")) {
        g_proto_split = value != 0;
    } else if (!strcmp(key, "force_imad")) {
        g_force_imad = value != 0;
    } else if (!strcmp(key, "algo")) {
        if (value < 0 || value > 2) return set_err(PFW_ERR_INVALID, "algo: 0 auto, 1 rule scan, 2 match sets");
        g_algo = (int)value;
    } else if (!strcmp(key, "matchset")) {
        g_matchset = value != 0;
    } else if (!strcmp(key, "matchset_budget_mb")) {
        if (value < 0) return set_err(PFW_ERR_INVALID, "matchset_budget_mb must be >= 0");
        g_ms_budget_mb = value;
    } else if (!strcmp(key, "ms_words")) {
        if (value != 1 && value != 2 && value != 4) return set_err(PFW_ERR_INVALID, "ms_words: 1, 2 or 4");
        g_ms_words = (int)value;
    } else if (!strcmp(key, "count_blocks")) {
        g_count_blocks = value != 0;
    } else if (!strcmp(key, "ms_compress")) {
        if (value < 0 || value > 2) return set_err(PFW_ERR_INVALID, "ms_compress: 0 off, 1 on, 2 auto");
        g_ms_compress = (int)value;
    } else if (!strcmp(key, "ms_summary")) {
        if (value < 0 || value > 2) return set_err(PFW_ERR_INVALID, "ms_summary: 0 off, 1 on, 2 auto");
        g_ms_summary = (int)value;
    } else if (!strcmp(key, "ms_group")) {
        if (value != 0 && value != 8 && value != 16 && value != 32)
            return set_err(PFW_ERR_INVALID, "ms_group: 0 (auto), 8, 16 or 32");
        g_ms_group = (int)value;
    } else if (!strcmp(key, "ms_lean_sum")) {
        if (value < 0 || value > 2) return set_err(PFW_ERR_INVALID, "ms_lean_sum: 0 off, 1 on, 2 on at 4 blocks per SM");
        g_ms_lean_sum = (int)value;
    } else if (!strcmp(key, "ms_lean_cmp")) {
        if (value < 0 || value > 3)
            return set_err(PFW_ERR_INVALID, "ms_lean_cmp: 0 off, 1 8-lane, 2 4-lane groups, 3 8-lane with u16 parked indices");
        g_ms_lean_cmp = (int)value;
    } else if (!strcmp(key, "ms_lean")) {
        if (value < 0 || value > 6)
            return set_err(PFW_ERR_INVALID, "ms_lean: 0 general kernel, 1 lean (8-lane groups), 2 lean (4-lane "
                                            "groups, 256-bit loads), 3 auto, 4 lean (4-lane groups, 512-rule "
                                            "steps), 5 lean (8-lane groups, 6 blocks per SM), 6 lean (64-packet batches)");
        g_ms_lean = (int)value;
    } else {
        return set_err(PFW_ERR_INVALID, "unknown tuning key '%s'", key);
    }
    return PFW_OK;
}

int pfw_ruleset_create(int device, int64_t n, const uint8_t *proto, const uint32_t *src_base,
                       const uint32_t *src_mask, const uint16_t *sport_lo, const uint16_t *sport_hi,
                       const uint32_t *dst_base, const uint32_t *dst_mask, const uint16_t *dport_lo,
                       const uint16_t *dport_hi, const uint8_t *accept, pfw_ruleset_t *out) {
    if (!out) return set_err(PFW_ERR_INVALID, "null output handle");
    *out = nullptr;
    if (n < 0 || n > PFW_MAX_RULES) return set_err(PFW_ERR_INVALID, "rule count %lld out of range", (long long)n);
    if (n > 0 && (!proto || !src_base || !src_mask || !sport_lo || !sport_hi || !dst_base ||
                  !dst_mask || !dport_lo || !dport_hi || !accept))
        return set_err(PFW_ERR_INVALID, "null rule column");
    // CIDR masks only (model.py:108-114): both encodings -- the range test
    // ip - base <= ~mask and the match-set interval [base, base | ~mask] --
    // equal the reference's (ip & mask) == base exactly for prefix masks
    for (int64_t r = 0; r < n; r++) {
        const uint32_t hs = ~src_mask[r], hd = ~dst_mask[r];
        if ((hs & (hs + 1u)) || (hd & (hd + 1u)))
            return set_err(PFW_ERR_INVALID, "rule %lld: %s mask 0x%08x is not a prefix mask", (long long)r,
                           (hs & (hs + 1u)) ? "src" : "dst", (hs & (hs + 1u)) ? src_mask[r] : dst_mask[r]);
    }
    int ndev = pfw_device_count();
    if (device < 0 || device >= ndev)
        return set_err(PFW_ERR_CUDA, "CUDA device %d not available (%d visible)", device, ndev);
    DeviceGuard g(device);
    if (!g.ok) return set_err(PFW_ERR_CUDA, "cudaSetDevice(%d) failed", device);

    NvtxRange nv("pfw_ruleset_create: pack + upload + match sets");
    pfw_ruleset *h = new pfw_ruleset();
    h->device = device;
    h->n = n;
    // pad: one full max-size stage (8 * 32 rules) past the last 32-aligned row
    h->rpad = ((n + 31) / 32) * 32 + 8 * 32;
    std::vector<uint32_t> host((size_t)NF * h->rpad);
    std::vector<uint8_t> acc((size_t)h->rpad, 0);
    for (int64_t r = 0; r < h->rpad; r++) {
        uint32_t w[NF];
        bool never = r >= n;
        if (!never) {
            const uint32_t sb = src_base[r], sm = src_mask[r], db = dst_base[r], dm = dst_mask[r];
            // (ip & mask) == base can only hold if base has no bits outside mask
            if ((sb & ~sm) || (db & ~dm)) never = true;
            if (sport_lo[r] > sport_hi[r] || dport_lo[r] > dport_hi[r]) never = true;
            w[F_SRC_NLO] = 0u - sb;
            w[F_SRC_W] = ~sm;
            w[F_DST_NLO] = 0u - db;
            w[F_DST_W] = ~dm;
            const uint32_t slo = sport_lo[r], shi = sport_hi[r], dlo = dport_lo[r], dhi = dport_hi[r];
            uint32_t loA, widA;
            float c1, c2;
            if (proto[r] == 0) {  // Protocol.ANY (model.py:68): A2 = sport<<8 | proto
                c1 = 0.f, c2 = 1.f;
                loA = slo << 8;
                widA = ((shi << 8) | 0xFFu) - loA;
            } else {              // concrete: A = proto<<16 | sport
                c1 = 1.f, c2 = 0.f;
                loA = ((uint32_t)proto[r] << 16) | slo;
                widA = shi - slo;
            }
            const uint32_t loB = dlo << 8, widB = ((dhi << 8) | 0xFFu) - loB;
            w[F_A_C1] = f2u(c1);
            w[F_A_C2] = f2u(c2);
            w[F_A_NLO] = f2u(-(float)loA);
            w[F_A_W] = f2u((float)widA);
            w[F_B_NLO] = f2u(-(float)loB);
            w[F_B_W] = f2u((float)widB);
            acc[r] = accept[r] ? 1 : 0;
        }
        if (never) {
            for (int f = 0; f < NF; f++) w[f] = 0;
            w[F_B_NLO] = NEVER_B_NLO;
            w[F_B_W] = NEVER_B_W;
        }
        for (int f = 0; f < NF; f++) host[(size_t)f * h->rpad + r] = w[f];
    }
    cudaError_t e = cudaMalloc(&h->d_rules, host.size() * 4);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_accept, acc.size());
    if (e == cudaSuccess) e = cudaMemcpy(h->d_rules, host.data(), host.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_accept, acc.data(), acc.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess && n > 0) {
        // protocol-split chains: one per concrete protocol named by a rule,
        // plus the ANY-only chain for every other protocol
        bool named[256] = {};
        for (int64_t r = 0; r < n; r++) named[proto[r]] = true;
        std::vector<int> protos;
        for (int v = 1; v < 256; v++)
            if (named[v]) protos.push_back(v);
        uint8_t lut[256];
        const int any_chain = (int)protos.size();
        for (int v = 0; v < 256; v++) lut[v] = (uint8_t)any_chain;
        for (size_t c = 0; c < protos.size(); c++) lut[protos[c]] = (uint8_t)c;
        h->chains.resize(protos.size() + 1);
        for (size_t c = 0; c <= protos.size() && e == cudaSuccess; c++) {
            pfw_ruleset::Chain &ch = h->chains[c];
            const int v = c < protos.size() ? protos[c] : -1;
            for (int64_t r = 0; r < n; r++)
                if (proto[r] == 0 || (int)proto[r] == v) ch.orig.push_back((uint32_t)r);
            ch.n = (int64_t)ch.orig.size();
            ch.rpad = ((ch.n + 31) / 32) * 32 + 8 * 32;
            std::vector<uint32_t> tab((size_t)NF * ch.rpad);
            std::vector<uint32_t> orig_pad((size_t)ch.rpad, 0);
            for (int64_t k = 0; k < ch.rpad; k++) {
                const int64_t r = k < ch.n ? (int64_t)ch.orig[(size_t)k] : n;  // n..: never-match pad row
                for (int f = 0; f < NF; f++) tab[(size_t)f * ch.rpad + k] = host[(size_t)f * h->rpad + r];
                orig_pad[(size_t)k] = k < ch.n ? ch.orig[(size_t)k] : 0u;
                // every packet scanned against this chain has protocol v, and
                // every rule in it is ANY or v: the protocol test is implied, so
                // concrete rules take the protocol-free sport form (A2 word)
                const bool live = k < ch.n && tab[(size_t)F_B_NLO * ch.rpad + k] != NEVER_B_NLO;
                if (live && proto[r] != 0) {
                    const uint32_t slo = sport_lo[r], shi = sport_hi[r];
                    const uint32_t loA = slo << 8, widA = ((shi << 8) | 0xFFu) - loA;
                    tab[(size_t)F_A_C1 * ch.rpad + k] = f2u(0.f);
                    tab[(size_t)F_A_C2 * ch.rpad + k] = f2u(1.f);
                    tab[(size_t)F_A_NLO * ch.rpad + k] = f2u(-(float)loA);
                    tab[(size_t)F_A_W * ch.rpad + k] = f2u((float)widA);
                }
            }
            e = cudaMalloc(&ch.d_rules, tab.size() * 4);
            if (e == cudaSuccess) e = cudaMalloc(&ch.d_orig, orig_pad.size() * 4);
            if (e == cudaSuccess) e = cudaMemcpy(ch.d_rules, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice);
            if (e == cudaSuccess) e = cudaMemcpy(ch.d_orig, orig_pad.data(), orig_pad.size() * 4, cudaMemcpyHostToDevice);
        }
        if (e == cudaSuccess) e = cudaMalloc(&h->d_lut, 256);
        if (e == cudaSuccess) e = cudaMemcpy(h->d_lut, lut, 256, cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) {
        const int rc = ms_create(h, proto, src_base, src_mask, sport_lo, sport_hi, dst_base, dst_mask, dport_lo,
                                 dport_hi);
        if (rc != PFW_OK) {
            pfw_ruleset_destroy(h);
            return rc;
        }
    }
    if (e != cudaSuccess) {
        const int code = e == cudaErrorMemoryAllocation ? PFW_ERR_NOMEM : PFW_ERR_CUDA;
        pfw_ruleset_destroy(h);
        return set_err(code, "ruleset upload failed: %s", cudaGetErrorString(e));
    }
    *out = h;
    return PFW_OK;
}

int pfw_ruleset_destroy(pfw_ruleset_t h) {
    if (!h) return PFW_OK;
    DeviceGuard g(h->device);
    if (h->d_rules) cudaFree(h->d_rules);
    if (h->d_accept) cudaFree(h->d_accept);
    if (h->d_ws) cudaFree(h->d_ws);
    if (h->h_stage) cudaFreeHost(h->h_stage);
    if (h->h_small) cudaFreeHost(h->h_small);
    free_ws(h->ws);
    if (h->d_peers) cudaFree(h->d_peers);
    for (auto &ch : h->chains) {
        if (ch.d_rules) cudaFree(ch.d_rules);
        if (ch.d_orig) cudaFree(ch.d_orig);
    }
    if (h->d_lut) cudaFree(h->d_lut);
    ms_free(h->ms);
    free_ws(h->ws_e2e[0]);
    free_ws(h->ws_e2e[1]);
    for (auto &st : h->streams)
        if (st) cudaStreamDestroy(st);
    for (auto &ev : h->events)
        if (ev) cudaEventDestroy(ev);
    delete h;
    return PFW_OK;
}

int64_t pfw_ruleset_size(pfw_ruleset_t h) { return h ? h->n : -1; }
int pfw_ruleset_device(pfw_ruleset_t h) { return h ? h->device : -1; }
int64_t pfw_ruleset_matchset_bytes(pfw_ruleset_t h) { return h && h->ms ? (int64_t)h->ms->bytes : 0; }

int pfw_ruleset_info(pfw_ruleset_t h, const char *key, int64_t *value) {
    if (!h || !key || !value) return set_err(PFW_ERR_INVALID, "null argument");
    const MatchSet *m = h->ms;
    if (!strcmp(key, "matchset_bytes")) *value = m ? (int64_t)m->bytes : 0;
    else if (!strcmp(key, "compressed")) *value = m && m->cmp ? 1 : 0;
    else if (!strcmp(key, "summaries")) *value = m && m->use_sum && m->sw > 0 ? 1 : 0;
    else if (!strcmp(key, "index_base")) *value = h->index_base;
    else return set_err(PFW_ERR_INVALID, "unknown ruleset info key '%s'", key);
    return PFW_OK;
}

int pfw_ruleset_set_shard(pfw_ruleset_t h, int64_t index_base, int64_t total) {
    if (!h) return set_err(PFW_ERR_INVALID, "null ruleset handle");
    if (index_base < 0 || total < 0 || index_base + h->n > total || total > PFW_MAX_RULES)
        return set_err(PFW_ERR_INVALID, "shard [%lld, %lld) outside a ruleset of %lld rules",
                       (long long)index_base, (long long)(index_base + h->n), (long long)total);
    h->index_base = index_base;
    h->total = total;
    return PFW_OK;
}

int pfw_pack_packets_host(int64_t n, const uint8_t *proto, const uint32_t *src_ip,
                          const uint16_t *src_port, const uint32_t *dst_ip,
                          const uint16_t *dst_port, void *h_out) {
    if (n < 0) return set_err(PFW_ERR_INVALID, "negative packet count");
    if (n == 0) return PFW_OK;
    if (!proto || !src_ip || !src_port || !dst_ip || !dst_port || !h_out)
        return set_err(PFW_ERR_INVALID, "null packet column");
    uint32_t *o = static_cast<uint32_t *>(h_out);
    for (int64_t i = 0; i < n; i++) {
        o[4 * i + 0] = src_ip[i];
        o[4 * i + 1] = dst_ip[i];
        o[4 * i + 2] = ((uint32_t)src_port[i] << 16) | dst_port[i];
        o[4 * i + 3] = proto[i];
    }
    return PFW_OK;
}

int pfw_scan_range(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts, int64_t n,
                   uint32_t *d_first, uint32_t *d_comps, uint8_t *d_verdict, uint64_t *d_stats,
                   void *stream) {
    return launch_scan(h, MODE_WRITE, lo, hi, d_pkts, n, d_first, d_comps, d_verdict, d_stats,
                       (cudaStream_t)stream);
}

int pfw_scan_range_columns(pfw_ruleset_t h, int64_t lo, int64_t hi, const uint8_t *d_proto,
                           const uint32_t *d_src_ip, const uint16_t *d_src_port, const uint32_t *d_dst_ip,
                           const uint16_t *d_dst_port, int64_t n, uint32_t *d_first, uint32_t *d_comps,
                           uint8_t *d_verdict, uint64_t *d_stats, void *stream) {
    const PacketCols c{d_proto, d_src_ip, d_src_port, d_dst_ip, d_dst_port};
    return launch_scan(h, MODE_WRITE, lo, hi, nullptr, n, d_first, d_comps, d_verdict, d_stats,
                       (cudaStream_t)stream, nullptr, nullptr, &c);
}

int pfw_scan_partition_accumulate(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts,
                                  int64_t n, uint32_t *d_first, uint32_t *d_comps,
                                  uint64_t *d_stats, void *stream) {
    return launch_scan(h, MODE_ACC, lo, hi, d_pkts, n, d_first, d_comps, nullptr, d_stats,
                       (cudaStream_t)stream);
}

int pfw_scan_fused_min(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts, int64_t n,
                       uint32_t *const *h_peer_first, uint32_t *const *h_peer_comps,
                       const int64_t *h_peer_cap, int npeers, int scatter, uint64_t *d_stats, void *stream) {
    if (!h) return set_err(PFW_ERR_INVALID, "null ruleset handle");
    if (npeers < 1 || npeers > MAX_PEERS) return set_err(PFW_ERR_INVALID, "npeers must be in 1..%d", MAX_PEERS);
    if (!h_peer_first || !h_peer_cap) return set_err(PFW_ERR_INVALID, "null peer table");
    if (n < 0) return set_err(PFW_ERR_INVALID, "negative packet count %lld", (long long)n);
    for (int i = 0; i < npeers; i++) {
        if (!h_peer_first[i] || (h_peer_comps && !h_peer_comps[i]))
            return set_err(PFW_ERR_INVALID, "null peer buffer %d", i);
        // rank i receives its shard of n (scatter) or all n packets: its
        // buffers must hold them, or the atomics would land past their end
        const int64_t need = scatter ? n / npeers + (i < n % npeers ? 1 : 0) : n;
        if (h_peer_cap[i] < need)
            return set_err(PFW_ERR_INVALID, "peer %d buffer holds %lld packets, the call needs %lld", i,
                           (long long)h_peer_cap[i], (long long)need);
    }
    if (n == 0) return PFW_OK;
    DeviceGuard g(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (!h->d_peers) CUDA_TRY(cudaMalloc(&h->d_peers, 2 * MAX_PEERS * sizeof(uint32_t *)));
    uint32_t *tab[2 * MAX_PEERS] = {};
    for (int i = 0; i < npeers; i++) {
        tab[i] = h_peer_first[i];
        tab[MAX_PEERS + i] = h_peer_comps ? h_peer_comps[i] : nullptr;
    }
    CUDA_TRY(cudaMemcpyAsync(h->d_peers, tab, sizeof tab, cudaMemcpyHostToDevice, st));
    // the table is read by the kernel later on the same stream; keep the host
    // copy alive until the copy has been issued (pageable -> staged now)
    ScanParams peer{};
    peer.peer_first = h->d_peers;
    peer.peer_comps = h_peer_comps ? h->d_peers + MAX_PEERS : nullptr;
    peer.npeers = npeers;
    peer.scatter = scatter ? 1 : 0;
    return launch_scan(h, MODE_PEER, lo, hi, d_pkts, n, nullptr, nullptr, nullptr, d_stats, st, nullptr,
                       &peer);
}

int pfw_peer_enable(int device, int peer) {
    const int ndev = pfw_device_count();
    if (device < 0 || device >= ndev || peer < 0 || peer >= ndev)
        return set_err(PFW_ERR_INVALID, "device %d / peer %d outside the %d visible devices", device, peer, ndev);
    if (device == peer) return PFW_OK;
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return set_err(PFW_ERR_CUDA, "device %d cannot access device %d's memory (no P2P)", device, peer);
    DeviceGuard g(device);
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return PFW_OK;
    }
    if (e != cudaSuccess) return set_err(PFW_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", device, peer,
                                         cudaGetErrorString(e));
    return PFW_OK;
}

int pfw_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// cudaIpcGetMemHandle exports the whole allocation that contains d_ptr; a
// caching allocator (torch) hands out pointers inside larger blocks, so the
// byte offset of d_ptr from the allocation base travels with the handle.
// The base comes from the driver's cuMemGetAddressRange, fetched through the
// runtime so that libpfw.so does not link libcuda (it must load without a GPU).
int pfw_ipc_get_handle(const void *d_ptr, void *out, uint64_t *offset) {
    if (!d_ptr || !out || !offset) return set_err(PFW_ERR_INVALID, "null pointer");
    typedef int (*range_fn)(unsigned long long *, size_t *, unsigned long long);
    static range_fn get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess)
            return set_err(PFW_ERR_CUDA, "cuMemGetAddressRange not available");
        get_range = (range_fn)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (unsigned long long)(uintptr_t)d_ptr) != 0)
        return set_err(PFW_ERR_CUDA, "cuMemGetAddressRange failed for %p", d_ptr);
    cudaIpcMemHandle_t hd;
    CUDA_TRY(cudaIpcGetMemHandle(&hd, const_cast<void *>(d_ptr)));
    memcpy(out, &hd, sizeof hd);
    *offset = (uint64_t)((uintptr_t)d_ptr - (uintptr_t)base);
    return PFW_OK;
}

int pfw_ipc_open(int device, const void *handle, void **out_base) {
    if (!handle || !out_base) return set_err(PFW_ERR_INVALID, "null pointer");
    DeviceGuard g(device);
    cudaIpcMemHandle_t hd;
    memcpy(&hd, handle, sizeof hd);
    CUDA_TRY(cudaIpcOpenMemHandle(out_base, hd, cudaIpcMemLazyEnablePeerAccess));
    return PFW_OK;
}

int pfw_ipc_close(int device, void *ptr) {
    if (!ptr) return PFW_OK;
    DeviceGuard g(device);
    CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return PFW_OK;
}

int pfw_scan_partitions(pfw_ruleset_t h, int64_t nodes, const void *d_pkts, int64_t n, uint32_t *d_first,
                        uint32_t *d_comps, uint64_t *d_stats, void *stream) {
    if (!h) return set_err(PFW_ERR_INVALID, "null ruleset handle");
    if (nodes < 1) return set_err(PFW_ERR_INVALID, "nodes must be >= 1, got %lld", (long long)nodes);
    if (n < 0) return set_err(PFW_ERR_INVALID, "negative packet count %lld", (long long)n);
    if (n > 0xFFFFFFFFll) return set_err(PFW_ERR_INVALID, "more than 2^32-1 packets in one call");
    if (n == 0) return PFW_OK;
    if (!d_pkts || !d_first || !d_comps) return set_err(PFW_ERR_INVALID, "null packet or output pointer");
    const cudaStream_t st = (cudaStream_t)stream;
    const int64_t R = h->n;
    // the non-empty partitions of partition_bounds(R, nodes) are partition_bounds(R, min(nodes, R))
    const int64_t parts = std::min<int64_t>(nodes, std::max<int64_t>(R, 1));
    NvtxRange nv("pfw scan (all partitions)");
    DeviceGuard g(h->device);
    if (!g.ok) return set_err(PFW_ERR_CUDA, "cudaSetDevice(%d) failed", h->device);
    // one accumulate launch per partition (a one-launch walk of every
    // partition per packet measured no faster: the steps dominate)
    int rc = pfw_accumulator_init(n, d_first, d_comps, stream);
    if (rc != PFW_OK) return rc;
    const int64_t q = R / parts, r = R % parts;
    for (int64_t j = 0, lo = 0; j < parts && R > 0; j++) {
        const int64_t hi = lo + q + (j < r ? 1 : 0);
        rc = launch_scan(h, MODE_ACC, lo, hi, d_pkts, n, d_first, d_comps, nullptr, d_stats, st);
        if (rc != PFW_OK) return rc;
        lo = hi;
    }
    return PFW_OK;
}

int pfw_accumulator_init(int64_t n, uint32_t *d_first, uint32_t *d_comps, void *stream) {
    if (n < 0 || (n > 0 && !d_first)) return set_err(PFW_ERR_INVALID, "bad accumulator arguments");
    if (n == 0) return PFW_OK;
    acc_init_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(n, d_first, d_comps);
    CUDA_TRY(cudaGetLastError());
    g_launches++;
    return PFW_OK;
}

int pfw_verdicts(pfw_ruleset_t h, const uint32_t *d_first, int64_t n, uint8_t *d_verdict,
                 void *stream) {
    if (!h || n < 0 || (n > 0 && (!d_first || !d_verdict)))
        return set_err(PFW_ERR_INVALID, "bad verdict arguments");
    if (h->total >= 0 && h->total != h->n)
        return set_err(PFW_ERR_INVALID, "verdicts of combined results need the whole ruleset's actions, not a "
                                        "shard of %lld of %lld rules", (long long)h->n, (long long)h->total);
    if (n == 0) return PFW_OK;
    DeviceGuard g(h->device);
    verdict_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(h->d_accept, d_first, n, d_verdict);
    CUDA_TRY(cudaGetLastError());
    g_launches++;
    return PFW_OK;
}

int pfw_combine_min(const uint32_t *d_rows, int64_t rows, int64_t n, uint32_t *d_out, void *stream) {
    if (rows < 0 || n < 0 || (n > 0 && (!d_out || (rows > 0 && !d_rows))))
        return set_err(PFW_ERR_INVALID, "bad combine arguments");
    if (n == 0) return PFW_OK;
    combine_min_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(d_rows, rows, n, d_out);
    CUDA_TRY(cudaGetLastError());
    g_launches++;
    return PFW_OK;
}

// Host buffers the DMA engines can read / write directly (pinned or
// registered, or managed); anything else is pageable and goes through the
// handle's pinned staging ring.
static double host_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static bool host_is_pinned(const void *p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged || a.type == cudaMemoryTypeDevice;
}

static int classify_host_impl(pfw_ruleset_t h, const void *h_pkts, const PacketCols *hc, int64_t n,
                              uint32_t *h_first, uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk,
                              uint32_t flags = 0, int64_t nodes = 0, uint32_t *h_comps = nullptr) {
    // Three-stage pipeline over E2E_SLOTS buffer slots:
    //   copy-in stream   H2D chunk k into slot k%S     (waits: scan k-S done)
    //   compute streams  scan chunk k on stream k%2    (waits: H2D k done); two
    //                    streams let chunk k+1's first pass fill the SMs
    //                    while chunk k's small late passes finish
    //   copy-out stream  D2H results of chunk k        (waits: scan k done)
    // so H2D of later chunks, the scans and D2H of earlier chunks all overlap.
    // Pageable caller buffers are staged through a pinned ring of the same S
    // slots by the host thread pool (HostPool): chunk k's columns are copied
    // into pinned memory while the GPU copies / scans earlier chunks, and a
    // chunk's results are copied out once its D2H has landed -- DMA from
    // pageable memory would otherwise stage synchronously and serialise the
    // pipeline.
    if (!h) return set_err(PFW_ERR_INVALID, "null ruleset handle");
    if (n < 0) return set_err(PFW_ERR_INVALID, "negative packet count");
    if (h_stats) h_stats[0] = h_stats[1] = 0;
    if (n == 0) return PFW_OK;
    if ((!h_pkts && !hc) || !h_first) return set_err(PFW_ERR_INVALID, "null host buffer");
    if (nodes < 0) return set_err(PFW_ERR_INVALID, "nodes must be >= 0");
    if (nodes > 0 && h->index_base != 0)
        return set_err(PFW_ERR_INVALID, "the partitioned e2e path needs a whole ruleset, not a rule shard");
    if (chunk <= 0) chunk = 1 << 23;
    // at least ~8 chunks per call (>= 256K packets each), so that smaller
    // batches pipeline too: a single chunk runs copy-in, scan and copy-out
    // one after the other
    {
        int64_t c8 = n / 8;
        if (c8 < (1 << 18)) c8 = 1 << 18;
        if (chunk > c8) chunk = c8;
    }
    if (chunk > n) chunk = n;
    DeviceGuard g(h->device);
    if (!g.ok) return set_err(PFW_ERR_CUDA, "cudaSetDevice(%d) failed", h->device);
    NvtxRange nv("pfw_classify_host: H2D / scan / D2H pipeline");
    constexpr int S = E2E_SLOTS;
    // which caller buffers need staging (inputs: records or the 5 columns)
    const void *in_ptr[5] = {h_pkts, nullptr, nullptr, nullptr, nullptr};
    size_t in_w[5] = {16, 0, 0, 0, 0};  // bytes per packet of each input buffer
    int nin = 1;
    if (hc) {
        const void *q[5] = {hc->src, hc->dst, hc->sport, hc->dport, hc->proto};
        const size_t w[5] = {4, 4, 2, 2, 1};
        for (int i = 0; i < 5; i++) in_ptr[i] = q[i], in_w[i] = w[i];
        nin = 5;
    }
    bool stage_in[5] = {}, any_in = false;
    for (int i = 0; i < nin; i++) any_in |= stage_in[i] = !host_is_pinned(in_ptr[i]);
    const bool stage_first = !host_is_pinned(h_first);
    const bool stage_verd = h_verdict && !host_is_pinned(h_verdict);
    const bool stage_comps = h_comps && !host_is_pinned(h_comps);
    const bool stage_out = stage_first || stage_verd || stage_comps;
    // slot: packets (16B records, or 13B of columns) + first 4B + verdict 1B
    // (+ comparisons 4B for the partitioned models)
    const size_t off_f = (size_t)chunk * 16, off_v = (size_t)chunk * 20, off_c = (((size_t)chunk * 21 + 15) / 16) * 16;
    const size_t slot = ((off_c + (nodes > 0 ? (size_t)chunk * 4 : 0) + 255) / 256) * 256;
    const size_t need = S * slot + 256;
    if (h->ws_bytes < need) {
        if (h->d_ws) cudaFree(h->d_ws);
        h->d_ws = nullptr;
        h->ws_bytes = 0;
        CUDA_TRY(cudaMalloc(&h->d_ws, need));
        h->ws_bytes = need;
    }
    if ((any_in || stage_out) && h->stage_bytes < S * slot) {
        if (h->h_stage) cudaFreeHost(h->h_stage);
        h->h_stage = nullptr;
        h->stage_bytes = 0;
        CUDA_TRY(cudaHostAlloc(&h->h_stage, S * slot, cudaHostAllocPortable));
        h->stage_bytes = S * slot;
    }
    for (auto &st : h->streams)
        if (!st) CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (auto &ev : h->events)
        if (!ev) CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaStream_t s_in = h->streams[0], s_out = h->streams[3];
    cudaEvent_t *ev_in = h->events, *ev_scan = h->events + S, *ev_out = h->events + 2 * S;
    char *ws = static_cast<char *>(h->d_ws);
    uint64_t *d_stats = reinterpret_cast<uint64_t *>(ws + S * slot);
    const uint32_t nomatch_out = (flags & PFW_HOST_FIRST_MINUS1) ? 0xFFFFFFFFu : PFW_NO_MATCH;
    // the scan of one chunk (m packets in the slot at `base`) on stream `sc`
    auto scan_chunk = [&](char *base, int64_t m, cudaStream_t sc, ScanWs *wsp) -> int {
        const uint4 *dp = reinterpret_cast<const uint4 *>(base);
        uint32_t *df = reinterpret_cast<uint32_t *>(base + off_f);
        uint8_t *dv = reinterpret_cast<uint8_t *>(base + off_v);
        uint32_t *dcm = reinterpret_cast<uint32_t *>(base + off_c);
        PacketCols dc{reinterpret_cast<const uint8_t *>(base + (size_t)chunk * 12), reinterpret_cast<const uint32_t *>(base),
                      reinterpret_cast<const uint16_t *>(base + (size_t)chunk * 8),
                      reinterpret_cast<const uint32_t *>(base + (size_t)chunk * 4),
                      reinterpret_cast<const uint16_t *>(base + (size_t)chunk * 10)};
        if (nodes == 0)
            return launch_scan(h, MODE_WRITE, 0, h->n, hc ? nullptr : dp, m, df, nullptr, h_verdict ? dv : nullptr,
                               h_stats ? d_stats : nullptr, sc, wsp, nullptr, hc ? &dc : nullptr, nomatch_out);
        // every node partition of partition_bounds(R, nodes) folded into the
        // chunk's first / comparisons (engines.py:349-369), then verdicts
        const int64_t R = h->n, parts = std::min<int64_t>(nodes, std::max<int64_t>(R, 1));
        acc_init_kernel<<<grid_for(m), 256, 0, sc>>>(m, df, dcm);
        g_launches++;
        const int64_t q = R / parts, r = R % parts;
        for (int64_t j = 0, lo = 0; j < parts && R > 0; j++) {
            const int64_t hi = lo + q + (j < r ? 1 : 0);
            const int rc2 = launch_scan(h, MODE_ACC, lo, hi, hc ? nullptr : dp, m, df, dcm, nullptr,
                                        h_stats ? d_stats : nullptr, sc, wsp, nullptr, hc ? &dc : nullptr);
            if (rc2 != PFW_OK) return rc2;
            lo = hi;
        }
        e2e_finish_kernel<<<grid_for(m), 256, 0, sc>>>(h->d_accept, df, h_verdict ? dv : nullptr, m, nomatch_out);
        g_launches++;
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? PFW_OK : set_err(PFW_ERR_CUDA, "e2e finish: %s", cudaGetErrorString(e));
    };
    // tiny batches (the serving case), any host memory: the inputs packed
    // into one pinned buffer in the slot's layout, ONE copy in, the scan, ONE
    // copy out of first / verdict / comparisons (+ the stats), one
    // synchronize; the host copies are a few KB
    if (n <= E2E_SMALL && n <= chunk) {
        NvtxRange nv0("pfw_classify_host: packed tiny batch");
        if (!h->h_small) CUDA_TRY(cudaHostAlloc(&h->h_small, (size_t)E2E_SMALL * 32 + 512, cudaHostAllocPortable));
        char *hsm = static_cast<char *>(h->h_small);
        const size_t in_bytes = hc ? (size_t)n * 13 : (size_t)n * 16;
        for (int i = 0; i < nin; i++)
            memcpy(hsm + (i == 0 || !hc ? 0 : (size_t)n * (i == 1 ? 4 : i == 2 ? 8 : i == 3 ? 10 : 12)), in_ptr[i],
                   (size_t)n * in_w[i]);
        cudaStream_t sc = h->streams[1];
        char *base = ws;
        if (h_stats) CUDA_TRY(cudaMemsetAsync(d_stats, 0, 16, sc));
        CUDA_TRY(cudaMemcpyAsync(base, hsm, in_bytes, cudaMemcpyHostToDevice, sc));
        int rc0 = scan_chunk(base, n, sc, &h->ws_e2e[0]);
        const size_t out_end = nodes > 0 ? off_c + (size_t)n * 4 : off_v + (size_t)n;
        const size_t stats_at = ((out_end + 15) / 16) * 16;
        if (rc0 == PFW_OK) {
            cudaError_t e = cudaMemcpyAsync(hsm + off_f, base + off_f, out_end - off_f, cudaMemcpyDeviceToHost, sc);
            if (e == cudaSuccess && h_stats) e = cudaMemcpyAsync(hsm + stats_at, d_stats, 16, cudaMemcpyDeviceToHost, sc);
            if (e != cudaSuccess) rc0 = set_err(PFW_ERR_CUDA, "tiny-batch copy failed: %s", cudaGetErrorString(e));
        }
        const cudaError_t es = cudaStreamSynchronize(sc);
        if (rc0 == PFW_OK && es != cudaSuccess)
            rc0 = set_err(PFW_ERR_CUDA, "cudaStreamSynchronize failed: %s", cudaGetErrorString(es));
        if (rc0 != PFW_OK) return rc0;
        memcpy(h_first, hsm + off_f, (size_t)n * 4);
        if (h_verdict) memcpy(h_verdict, hsm + off_v, (size_t)n);
        if (h_comps && nodes > 0) memcpy(h_comps, hsm + off_c, (size_t)n * 4);
        if (h_stats) memcpy(h_stats, hsm + stats_at, 16);
        return PFW_OK;
    }
    // one chunk, pinned buffers (small batches): copy in, scan and copy out
    // on one stream, one synchronize -- no events, no cross-stream waits
    if (n <= chunk && !any_in && !stage_out) {
        NvtxRange nv1("pfw_classify_host: single-stream small batch");
        cudaStream_t sc = h->streams[1];
        char *base = ws;
        if (h_stats) CUDA_TRY(cudaMemsetAsync(d_stats, 0, 16, sc));
        for (int i = 0; i < nin; i++)
            CUDA_TRY(cudaMemcpyAsync(base + (i == 0 || !hc ? 0 : (size_t)chunk * (i == 1 ? 4 : i == 2 ? 8 : i == 3 ? 10 : 12)),
                                     in_ptr[i], (size_t)n * in_w[i], cudaMemcpyHostToDevice, sc));
        int rc1 = scan_chunk(base, n, sc, &h->ws_e2e[0]);
        if (rc1 == PFW_OK) {
            cudaError_t e = cudaMemcpyAsync(h_first, base + off_f, (size_t)n * 4, cudaMemcpyDeviceToHost, sc);
            if (e == cudaSuccess && h_verdict)
                e = cudaMemcpyAsync(h_verdict, base + off_v, (size_t)n, cudaMemcpyDeviceToHost, sc);
            if (e == cudaSuccess && h_comps && nodes > 0)
                e = cudaMemcpyAsync(h_comps, base + off_c, (size_t)n * 4, cudaMemcpyDeviceToHost, sc);
            if (e == cudaSuccess && h_stats) e = cudaMemcpyAsync(h_stats, d_stats, 16, cudaMemcpyDeviceToHost, sc);
            if (e != cudaSuccess) rc1 = set_err(PFW_ERR_CUDA, "small-batch copy failed: %s", cudaGetErrorString(e));
        }
        const cudaError_t es = cudaStreamSynchronize(sc);  // (always: queued copies target the caller's buffers)
        if (rc1 == PFW_OK && es != cudaSuccess)
            rc1 = set_err(PFW_ERR_CUDA, "cudaStreamSynchronize failed: %s", cudaGetErrorString(es));
        return rc1;
    }
    if (h_stats) {
        CUDA_TRY(cudaMemsetAsync(d_stats, 0, 16, s_in));
        CUDA_TRY(cudaEventRecord(ev_in[0], s_in));  // ordered before every compute stream below
    }
    // Chunk schedule: ramp up (1/8, 1/4, 1/2 of the chunk) at the start and
    // down at the end, so the pipeline fills after a small first copy-in and
    // drains after a small last scan + copy-out (the fill / drain otherwise
    // cost a whole chunk each: ~10% of a 64Mi-packet call)
    std::vector<int64_t> sizes;
    {
        std::vector<int64_t> ramp;
        for (int64_t r = chunk / 8; r > 0 && r < chunk; r *= 2)  // (chunk < 8: no ramp)
            if (r >= (1 << 16)) ramp.push_back(r);
        int64_t rs = 0;
        for (int64_t r : ramp) rs += r;
        if (!ramp.empty() && n >= 2 * rs + 2 * chunk) {
            sizes = ramp;
            int64_t mid = n - 2 * rs;
            while (mid > 0) {
                const int64_t mm = mid < chunk ? mid : chunk;
                sizes.push_back(mm);
                mid -= mm;
            }
            sizes.insert(sizes.end(), ramp.rbegin(), ramp.rend());
        } else {
            for (int64_t c0 = 0; c0 < n; c0 += chunk) sizes.push_back(n - c0 < chunk ? n - c0 : chunk);
        }
    }
    const int64_t nchunks = (int64_t)sizes.size();
    std::vector<int64_t> starts((size_t)nchunks + 1, 0);
    for (int64_t k = 0; k < nchunks; k++) starts[(size_t)k + 1] = starts[(size_t)k] + sizes[(size_t)k];
    HostPool &pool = HostPool::get();
    char *hs = static_cast<char *>(h->h_stage);
    // slot layout (device and staging alike): inputs at [0, 16*chunk) -- records,
    // or columns src | dst | sport | dport | proto at 0, 4, 8, 10, 12 x chunk --,
    // first at 16*chunk, verdict at 20*chunk
    const size_t in_off[5] = {0, (size_t)chunk * 4, (size_t)chunk * 8, (size_t)chunk * 10, (size_t)chunk * 12};
    int64_t drained = 0;  // chunks whose staged results have been copied out
    // PFW_E2E_TRACE=1: per-call host-side timing of the staging path (stderr)
    static const bool trace = getenv("PFW_E2E_TRACE") != nullptr;
    double t_wait = 0.0, t_copy = 0.0;
    const double t_call = trace ? host_seconds() : 0.0;
    auto drain = [&](int64_t upto) -> cudaError_t {  // copy staged results of chunks < upto out
        for (; drained < upto; drained++) {
            const int sl = (int)(drained % S);
            const cudaError_t e = cudaEventSynchronize(ev_out[sl]);
            if (e != cudaSuccess) return e;
            const int64_t c0 = starts[(size_t)drained], m = sizes[(size_t)drained];
            char *base = hs + sl * slot;
            HostPool::Copy cps[3];
            int ncp = 0;
            if (stage_first) cps[ncp++] = HostPool::Copy{h_first + c0, base + off_f, (size_t)m * 4};
            if (stage_verd) cps[ncp++] = HostPool::Copy{h_verdict + c0, base + off_v, (size_t)m};
            if (stage_comps) cps[ncp++] = HostPool::Copy{h_comps + c0, base + off_c, (size_t)m * 4};
            pool.copy_many(cps, ncp);
        }
        return cudaSuccess;
    };
    int rc = PFW_OK;
    // inside the loop an error stops issuing work but never returns before
    // the streams are drained: copies already queued still target the
    // caller's host buffers
#define E2E_TRY(expr)                                                                       \
    {                                                                                       \
        const cudaError_t e2e_err_ = (expr);                                                \
        if (e2e_err_ != cudaSuccess) {                                                      \
            rc = set_err(PFW_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e2e_err_)); \
            break;                                                                          \
        }                                                                                   \
    }
    for (int64_t k = 0; k < nchunks && rc == PFW_OK; k++) {
        const int64_t c0 = starts[(size_t)k], m = sizes[(size_t)k];
        const int sl = (int)(k % S);
        cudaStream_t s_comp = h->streams[1 + (k & 1)];
        char *base = ws + sl * slot;
        char *sbase = hs + sl * slot;
        uint32_t *df = reinterpret_cast<uint32_t *>(base + off_f);
        uint8_t *dv = reinterpret_cast<uint8_t *>(base + off_v);
        uint32_t *dcm = reinterpret_cast<uint32_t *>(base + off_c);
        if (k >= S) E2E_TRY(cudaStreamWaitEvent(s_in, ev_scan[sl], 0));   // packets slot free
        if (any_in) {
            // the staging slot's previous H2D (chunk k - S) must have read it
            const double tw0 = trace ? host_seconds() : 0.0;
            if (k >= S) E2E_TRY(cudaEventSynchronize(ev_in[sl]));
            const double tw1 = trace ? host_seconds() : 0.0;
            HostPool::Copy cps[5];
            int ncp = 0;
            for (int i = 0; i < nin; i++)
                if (stage_in[i])
                    cps[ncp++] = HostPool::Copy{sbase + in_off[i],
                                                static_cast<const char *>(in_ptr[i]) + (size_t)c0 * in_w[i],
                                                (size_t)m * in_w[i]};
            pool.copy_many(cps, ncp);
            if (trace) {
                t_wait += tw1 - tw0;
                t_copy += host_seconds() - tw1;
            }
        }
        bool fail = false;
        for (int i = 0; i < nin; i++) {
            const char *src = stage_in[i] ? sbase + in_off[i]
                                          : static_cast<const char *>(in_ptr[i]) + (size_t)c0 * in_w[i];
            const cudaError_t e = cudaMemcpyAsync(base + in_off[i], src, (size_t)m * in_w[i],
                                                  cudaMemcpyHostToDevice, s_in);
            if (e != cudaSuccess) {
                rc = set_err(PFW_ERR_CUDA, "H2D copy failed: %s", cudaGetErrorString(e));
                fail = true;
                break;
            }
        }
        if (fail) break;
        E2E_TRY(cudaEventRecord(ev_in[sl], s_in));
        E2E_TRY(cudaStreamWaitEvent(s_comp, ev_in[sl], 0));
        if (k >= S) E2E_TRY(cudaStreamWaitEvent(s_comp, ev_out[sl], 0));  // result slot drained
        rc = scan_chunk(base, m, s_comp, &h->ws_e2e[k & 1]);
        if (rc != PFW_OK) break;
        E2E_TRY(cudaEventRecord(ev_scan[sl], s_comp));
        E2E_TRY(cudaStreamWaitEvent(s_out, ev_scan[sl], 0));
        // a staged output slot is reused by chunk k: chunk k - S's results
        // must have been copied out of it first
        if (stage_out) E2E_TRY(drain(k - S + 1 > 0 ? k - S + 1 : 0));
        E2E_TRY(cudaMemcpyAsync(stage_first ? reinterpret_cast<uint32_t *>(sbase + off_f) : h_first + c0,
                                df, m * 4, cudaMemcpyDeviceToHost, s_out));
        if (h_verdict)
            E2E_TRY(cudaMemcpyAsync(stage_verd ? reinterpret_cast<uint8_t *>(sbase + off_v) : h_verdict + c0,
                                    dv, m, cudaMemcpyDeviceToHost, s_out));
        if (h_comps && nodes > 0)
            E2E_TRY(cudaMemcpyAsync(stage_comps ? reinterpret_cast<uint32_t *>(sbase + off_c) : h_comps + c0,
                                    dcm, m * 4, cudaMemcpyDeviceToHost, s_out));
        E2E_TRY(cudaEventRecord(ev_out[sl], s_out));
        // copy out what has landed meanwhile (keeps the host busy while the
        // GPU works; never waits for the chunk just issued)
        if (stage_out && k >= 1) E2E_TRY(drain(k - 1 > drained ? k - 1 : drained));
    }
#undef E2E_TRY
    for (auto &st : h->streams) {
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess && rc == PFW_OK)
            rc = set_err(PFW_ERR_CUDA, "cudaStreamSynchronize failed: %s", cudaGetErrorString(e));
    }
    if (rc != PFW_OK) return rc;
    if (stage_out) {
        const cudaError_t e = drain(nchunks);
        if (e != cudaSuccess) return set_err(PFW_ERR_CUDA, "staged copy-out failed: %s", cudaGetErrorString(e));
    }
    if (h_stats) CUDA_TRY(cudaMemcpy(h_stats, d_stats, 16, cudaMemcpyDeviceToHost));
    if (trace)
        fprintf(stderr, "pfw e2e: n=%lld chunks=%lld stage_in=%d stage_out=%d call %.2f ms, slot waits %.2f ms, "
                        "staging copies %.2f ms (%d pool threads)\n", (long long)n, (long long)nchunks, (int)any_in,
                (int)stage_out, (host_seconds() - t_call) * 1e3, t_wait * 1e3, t_copy * 1e3,
                pool.threads());
    return PFW_OK;
}


int pfw_classify_host(pfw_ruleset_t h, const void *h_pkts, int64_t n, uint32_t *h_first,
                      uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk) {
    return classify_host_impl(h, h_pkts, nullptr, n, h_first, h_verdict, h_stats, chunk);
}

int pfw_classify_host_columns(pfw_ruleset_t h, const uint8_t *h_proto, const uint32_t *h_src_ip,
                              const uint16_t *h_src_port, const uint32_t *h_dst_ip,
                              const uint16_t *h_dst_port, int64_t n, uint32_t *h_first,
                              uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk) {
    if (n > 0 && (!h_proto || !h_src_ip || !h_src_port || !h_dst_ip || !h_dst_port))
        return set_err(PFW_ERR_INVALID, "null packet column");
    const PacketCols hc{h_proto, h_src_ip, h_src_port, h_dst_ip, h_dst_port};
    return classify_host_impl(h, nullptr, &hc, n, h_first, h_verdict, h_stats, chunk);
}

int pfw_classify_host_ex(pfw_ruleset_t h, const void *h_pkts, const uint8_t *h_proto, const uint32_t *h_src_ip,
                         const uint16_t *h_src_port, const uint32_t *h_dst_ip, const uint16_t *h_dst_port,
                         int64_t n, uint32_t *h_first, uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk,
                         uint32_t flags) {
    if (flags & ~(uint32_t)PFW_HOST_FIRST_MINUS1) return set_err(PFW_ERR_INVALID, "unknown flags 0x%x", flags);
    if (h_pkts) return classify_host_impl(h, h_pkts, nullptr, n, h_first, h_verdict, h_stats, chunk, flags);
    if (n > 0 && (!h_proto || !h_src_ip || !h_src_port || !h_dst_ip || !h_dst_port))
        return set_err(PFW_ERR_INVALID, "null packet column");
    const PacketCols hc{h_proto, h_src_ip, h_src_port, h_dst_ip, h_dst_port};
    return classify_host_impl(h, nullptr, &hc, n, h_first, h_verdict, h_stats, chunk, flags);
}

int pfw_classify_host_partitions(pfw_ruleset_t h, int64_t nodes, const void *h_pkts, const uint8_t *h_proto,
                                 const uint32_t *h_src_ip, const uint16_t *h_src_port, const uint32_t *h_dst_ip,
                                 const uint16_t *h_dst_port, int64_t n, uint32_t *h_first, uint32_t *h_comps,
                                 uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk, uint32_t flags) {
    if (flags & ~(uint32_t)PFW_HOST_FIRST_MINUS1) return set_err(PFW_ERR_INVALID, "unknown flags 0x%x", flags);
    if (nodes < 1) return set_err(PFW_ERR_INVALID, "nodes must be >= 1, got %lld", (long long)nodes);
    if (n > 0 && !h_comps) return set_err(PFW_ERR_INVALID, "null comparisons buffer");
    if (h_pkts) return classify_host_impl(h, h_pkts, nullptr, n, h_first, h_verdict, h_stats, chunk, flags, nodes, h_comps);
    if (n > 0 && (!h_proto || !h_src_ip || !h_src_port || !h_dst_ip || !h_dst_port))
        return set_err(PFW_ERR_INVALID, "null packet column");
    const PacketCols hc{h_proto, h_src_ip, h_src_port, h_dst_ip, h_dst_port};
    return classify_host_impl(h, nullptr, &hc, n, h_first, h_verdict, h_stats, chunk, flags, nodes, h_comps);
}

int pfw_generate_traffic(int device, uint64_t seed, int64_t n, int proto, uint32_t src_base,
                         int src_plen, uint32_t dst_base, int dst_plen, int sport_lo, int sport_hi,
                         int dport_lo, int dport_hi, void *d_out, void *stream) {
    return pfw_generate_traffic_at(device, seed, 0, n, proto, src_base, src_plen, dst_base, dst_plen,
                                   sport_lo, sport_hi, dport_lo, dport_hi, d_out, stream);
}

int pfw_generate_traffic_at(int device, uint64_t seed, int64_t first_packet, int64_t n, int proto,
                            uint32_t src_base, int src_plen, uint32_t dst_base, int dst_plen,
                            int sport_lo, int sport_hi, int dport_lo, int dport_hi, void *d_out,
                            void *stream) {
    if (n < 0 || first_packet < 0) return set_err(PFW_ERR_INVALID, "count and first_packet must be >= 0");
    if (proto <= 0 || proto > 255) return set_err(PFW_ERR_INVALID, "traffic protocol must be concrete (1..255)");
    if (src_plen < 0 || src_plen > 32 || dst_plen < 0 || dst_plen > 32)
        return set_err(PFW_ERR_INVALID, "prefix length outside 0..32");
    if (sport_lo < 0 || sport_hi > 65535 || sport_lo > sport_hi || dport_lo < 0 ||
        dport_hi > 65535 || dport_lo > dport_hi)
        return set_err(PFW_ERR_INVALID, "bad port range");
    if (first_packet > 0 && (((sport_hi - sport_lo + 1) & (sport_hi - sport_lo)) != 0 ||
                             ((dport_hi - dport_lo + 1) & (dport_hi - dport_lo)) != 0))
        return set_err(PFW_ERR_INVALID,
                       "first_packet > 0 needs power-of-two port spans (then every packet is exactly "
                       "4 draws and the stream position is known)");
    if (n == 0) return PFW_OK;
    if (!d_out) return set_err(PFW_ERR_INVALID, "null output");
    int ndev = pfw_device_count();
    if (device < 0 || device >= ndev) return set_err(PFW_ERR_CUDA, "CUDA device %d not available", device);
    DeviceGuard g(device);
    cudaStream_t st = (cudaStream_t)stream;
    NvtxRange nv("pfw_generate_traffic");

    GenParams gp{};
    gp.proto = (uint32_t)proto;
    const uint32_t smask = src_plen ? (uint32_t)(0xFFFFFFFFull << (32 - src_plen)) : 0u;
    const uint32_t dmask = dst_plen ? (uint32_t)(0xFFFFFFFFull << (32 - dst_plen)) : 0u;
    gp.src_base = src_base & smask;  // TrafficProfile subnets are normalised CidrMatchers
    gp.dst_base = dst_base & dmask;
    gp.sspan = 1ULL << (32 - src_plen);
    gp.dspan = 1ULL << (32 - dst_plen);
    gp.sp_lo = (uint32_t)sport_lo;
    gp.dp_lo = (uint32_t)dport_lo;
    gp.sp_n = (uint64_t)(sport_hi - sport_lo + 1);
    gp.dp_n = (uint64_t)(dport_hi - dport_lo + 1);
    {
        const uint64_t r1 = (0 - gp.sp_n) % gp.sp_n, r2 = (0 - gp.dp_n) % gp.dp_n;
        gp.sp_lim = r1 ? 0 - r1 : 0;
        gp.dp_lim = r2 ? 0 - r2 : 0;
    }
    // jump matrices: per-thread jump = M^(4*GEN_PER_THREAD); per-block = M^(4*GEN_PER_BLOCK)
    static std::mutex mu;
    static bool ready = false;
    static Mat64 jblock;
    static uint64_t jthread[GEN_LOG_BLOCK][64];
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!ready) {
            Mat64 m = mat_step();
            Mat64 jt = mat_pow(m, 4ULL * GEN_PER_THREAD);
            for (int b = 0; b < GEN_LOG_BLOCK; b++) {
                memcpy(jthread[b], jt.c, sizeof jt.c);
                jt = mat_mul(jt, jt);
            }
            jblock = mat_pow(m, 4ULL * GEN_PER_BLOCK);
            ready = true;
        }
    }
    static thread_local int uploaded_dev_mask = 0;
    if (!(uploaded_dev_mask & (1 << device))) {
        CUDA_TRY(cudaMemcpyToSymbol(c_jump, jthread, sizeof jthread));
        uploaded_dev_mask |= 1 << device;
    }

    struct Scratch {  // freed on every return path
        uint64_t *d_state = nullptr;
        unsigned long long *d_rej = nullptr;
        ~Scratch() {
            if (d_state) cudaFree(d_state);
            if (d_rej) cudaFree(d_rej);
        }
    } sc;
    uint64_t *&d_state = sc.d_state;
    unsigned long long *&d_rej = sc.d_rej;
    int64_t start = 0;
    Mat64 m1 = mat_step();
    uint64_t x = host_seed_state(seed);  // state before packet `start`
    if (first_packet > 0) x = matvec(mat_pow(m1, 4ULL * (uint64_t)first_packet).c, x);
    int rc = PFW_OK;
    int rounds = 0;
    while (start < n) {
        const int64_t rem = n - start;
        const int64_t nblocks = (rem + GEN_PER_BLOCK - 1) / GEN_PER_BLOCK;
        std::vector<uint64_t> states((size_t)nblocks);
        uint64_t s = x;
        for (int64_t b = 0; b < nblocks; b++) {
            states[(size_t)b] = s;
            s = matvec(jblock.c, s);
        }
        if (d_state) cudaFree(d_state);
        d_state = nullptr;
        CUDA_TRY(cudaMalloc(&d_state, states.size() * 8));
        if (!d_rej) CUDA_TRY(cudaMalloc(&d_rej, 8));
        CUDA_TRY(cudaMemcpyAsync(d_state, states.data(), states.size() * 8, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemsetAsync(d_rej, 0xFF, 8, st));
        gen_kernel<<<(unsigned)nblocks, GEN_BLOCK, 0, st>>>(gp, d_state, start, n,
                                                           static_cast<uint4 *>(d_out), d_rej);
        CUDA_TRY(cudaGetLastError());
        g_launches++;
        unsigned long long rej = 0;
        CUDA_TRY(cudaMemcpyAsync(&rej, d_rej, 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (rej == ~0ULL) break;
        // A bounded draw was rejected inside packet `rej`: every packet before
        // it is exact.  Regenerate packet `rej` on the host with the exact
        // rejection loop (rng.py:54-62), then resume the device stream after it.
        if (++rounds > 1000000) { rc = set_err(PFW_ERR_GENERATION, "too many rejection repairs"); break; }
        uint64_t y = matvec(mat_pow(m1, 4ULL * (uint64_t)(rej - start)).c, x);
        uint4 v;
        v.x = gp.src_base + (uint32_t)host_randbelow(y, gp.sspan);
        const uint32_t sp = gp.sp_lo + (uint32_t)host_randbelow(y, gp.sp_n);
        v.y = gp.dst_base + (uint32_t)host_randbelow(y, gp.dspan);
        const uint32_t dp = gp.dp_lo + (uint32_t)host_randbelow(y, gp.dp_n);
        v.z = (sp << 16) | dp;
        v.w = gp.proto;
        CUDA_TRY(cudaMemcpyAsync(static_cast<uint4 *>(d_out) + rej, &v, 16, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        start = (int64_t)rej + 1;
        x = y;
    }
    return rc;
}

}  // extern "C"
