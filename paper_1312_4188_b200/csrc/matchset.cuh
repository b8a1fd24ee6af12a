// matchset.cuh -- the first-match scan over per-field match sets (included by
// pfw.cu inside its anonymous namespace).
//
// Each rule field accepts one interval of its value domain: a CIDR block
// [base, base | ~mask] (model.py:108-121), an inclusive port range [lo, hi]
// (model.py:144-145), a protocol value or all of them (model.py:222-230).
// The end points of all rules' intervals cut a field's domain into elementary
// intervals; inside one, every rule's field test has the same outcome.  Row i
// of a field's bitmap holds bit r = "rule r's test on this field holds on
// interval i" (rule r at word r/32, bit r%32).  A packet's first match in the
// window [lo, hi) (classifier.py:146-162) is the lowest set bit of the AND of
// its four rows -- src, dst, (protocol class, sport), dport; the protocol is
// folded into the sport rows, one block of rows per protocol class -- so the
// scan reads 128-byte lines of 1024 rules per warp step instead of testing
// rule by rule.  Results are the rule-by-rule scan's, bit for bit: the rows
// are built by the reference predicate itself, evaluated on each interval's
// first value.
//
// Layout in HBM (struct MatchSet): the four dimensions' rows in one
// allocation, rows x wp words each (wp = rules/32 rounded up to a whole step
// of 128 words, 512 bytes); optional block summaries (one bit per 1024-rule
// block per row); compressed rows above 16K rules (each (dimension, 1024-rule
// block) stores its distinct lines once, rows hold u16 line indices, a dense
// head array the first 8 blocks'); IP value -> interval through a 65536-entry
// table of 16-byte /16-block entries (boundary range + the first 6 boundaries'
// low halves) and the sorted boundaries; port value -> interval through a
// direct 65536-entry table; protocol -> class through a 256-entry table.  The
// lookup tables (~2.5 MB) and the rows' leading lines (where most first
// matches are) stay resident in L2 up to ~10K rules.
//
// Kernels: ms_lean_kernel (whole-table scans over plain rows: data / grid /
// oracle configs), ms_lean_cmp_kernel (compressed rows: function config),
// ms_lean_sum_kernel (block-summary candidate walk: adversarial config),
// ms_scan_kernel (general: windows, accumulate / fused-combine epilogues, the
// other shapes), plus the build kernels.  DESIGN.md section 3 has the shapes
// and their measurements.

constexpr int MS_BLOCK = 256;
#ifndef PFW_MS_MINB
#define PFW_MS_MINB 5  // resident blocks per SM the scan is register-limited to
#endif
#ifndef PFW_MS_MINB_SC
#define PFW_MS_MINB_SC 4  // the summary scan over compressed rows (two candidates per step)
#endif
#ifndef PFW_MS_PARK
#define PFW_MS_PARK 6  // compressed rows: blocks of line numbers parked per packet and dimension (1..8)
#endif
#ifndef PFW_MS_LPB
#define PFW_MS_LPB 1   // packets per lane per batch (batch = 32 * LPB packets per warp)
#endif
enum { MSD_SRC = 0, MSD_DST = 1, MSD_SPORT = 2, MSD_DPORT = 3 };

int g_matchset = 1;            // build match sets at ruleset creation
int g_algo = 0;                // 0 auto (match sets when built), 1 rule-by-rule scan, 2 match sets
int64_t g_ms_budget_mb = 0;    // device-memory budget for the tables (0 = a quarter of free memory)
int g_ms_group = 0;            // lanes per packet (8, 16, 32; 0 = by ruleset size): 32 / group packets in flight per warp
int g_ms_words = 4;            // words per lane per step: 32 * group * words rules per step
int g_ms_summary = 2;          // block summaries: 0 off, 1 on, 2 auto (built and used when they skip enough)
int g_ms_compress = 2;         // compressed rows: 0 off, 1 on, 2 auto (see ms_create)
// auto: compressed rows above this many rules.  Above it the plain rows'
// leading lines no longer stay in L2 (r2 sweep, 16Mi packets: plain 12.9 Gpps
// at 16K rules, 10.1 at 18K, 9.3 at 20K; compressed ~10.6 flat from 10K up)
constexpr int64_t MS_CMP_MIN_RULES = 16384;
constexpr double MS_SUM_KEEP_MAX = 0.75;  // auto: use summaries if a packet keeps < 75% of blocks
int g_ms_lean = 3;             // whole-table plain-row scans: 0 general kernel, 1 lean 8-lane groups, 2 lean 4-lane groups (256-bit loads), 3 auto
int g_count_blocks = 0;        // count the summary scan's block reads (pfw_read_counter "blocks_read")
int g_ms_lean_sum = 2;         // whole-table summary scans over compressed rows: lean candidate walk (0 general kernel, 1 at 5 / 2 at 4 blocks per SM)
int g_ms_lean_cmp = 3;         // whole-table scans over compressed rows: 0 general kernel, 1 lean 8-lane, 2 lean 4-lane, 3 lean 8-lane with u16 parked indices (<= MS_CP_BLOCKS blocks, else 1)
unsigned long long *g_counter_dev = nullptr;  // device of the first counting launch

struct MsBuildArgs {
    const uint32_t *base, *mask;  // IP fields
    const uint16_t *lo, *hi;      // port fields
    const uint8_t *proto;         // rule protocols (sport field)
    const uint32_t *vals;         // first value of each elementary interval
    const int *cls_proto;         // sport field: protocol of class c (-1: a protocol no rule names)
    int64_t n, wp, rows, ivl;     // rules, words per row, rows, intervals per class (sport)
    uint32_t *bits;
};

// One warp per (32-word group, row): lane = rule inside each word, one ballot
// per word, lane k keeps word k, one coalesced 128-byte store.  Consecutive
// warps share a word group, so the rule columns are L1 hits.
template <int D>
__global__ void __launch_bounds__(MS_BLOCK) ms_build_kernel(MsBuildArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t groups = a.wp / 32;
    for (int64_t t = gw; t < groups * a.rows; t += nw) {
        const int64_t g = t / a.rows, row = t - g * a.rows;
        uint32_t v;
        int pcl = -1;
        if (D == MSD_SPORT) {
            const int64_t c = row / a.ivl;
            v = __ldg(a.vals + (row - c * a.ivl));
            pcl = __ldg(a.cls_proto + c);
        } else {
            v = __ldg(a.vals + row);
        }
        uint32_t mine = 0;
#pragma unroll 4
        for (int k = 0; k < 32; k++) {
            const int64_t r = (g * 32 + k) * 32 + lane;
            bool m = false;
            if (r < a.n) {
                if (D == MSD_SRC || D == MSD_DST) {
                    m = (v & __ldg(a.mask + r)) == __ldg(a.base + r);         // model.py:119-121
                } else {
                    m = (uint32_t)__ldg(a.lo + r) <= v && v <= (uint32_t)__ldg(a.hi + r);  // model.py:144-145
                    if (D == MSD_SPORT) {
                        const int rp = __ldg(a.proto + r);                     // model.py:224-225
                        m = m && (rp == 0 || rp == pcl);
                    }
                }
            }
            const uint32_t b = __ballot_sync(0xFFFFFFFFu, m);
            if (lane == k) mine = b;
        }
        PFW_CHECK(row < a.rows && g * 32 + lane < a.wp);
        a.bits[row * a.wp + g * 32 + lane] = mine;
    }
}

// Summary rows: warp per (row, summary word j); lane k ORs block 32j+k's 32
// words (eight 16-byte loads) and one ballot forms the word.
__global__ void __launch_bounds__(MS_BLOCK) ms_sum_kernel(const uint32_t *bits, int64_t rows, int64_t wp,
                                                          int64_t sw, uint32_t *sum) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t blocks = wp / 32;
    for (int64_t t = gw; t < rows * sw; t += nw) {
        const int64_t row = t / sw, j = t - row * sw, blk = j * 32 + lane;
        uint32_t any = 0;
        if (blk < blocks) {
            const uint4 *q = reinterpret_cast<const uint4 *>(bits + row * wp + blk * 32);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint4 v = __ldg(q + k);
                any |= v.x | v.y | v.z | v.w;
            }
        }
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, any != 0u);
        if (lane == 0) sum[row * sw + j] = b;
    }
}

// Compressed rows: one descriptor per distinct line of (dimension, block).
struct MsLineDesc {
    uint32_t v;      // first value of the block-local interval
    uint32_t b;      // block (rules 1024 b .. 1024 b + 1023)
    uint16_t d, c;   // dimension, protocol class (sport)
};

// warp per line: lane = rule inside each word, one ballot per word (as
// ms_build_kernel, on the block's 1024 rules only)
__global__ void __launch_bounds__(MS_BLOCK) ms_line_kernel(const MsLineDesc *desc, int64_t nlines, int64_t n,
                                                           const uint32_t *sb, const uint32_t *sm,
                                                           const uint32_t *db, const uint32_t *dm,
                                                           const uint16_t *slo, const uint16_t *shi,
                                                           const uint16_t *dlo, const uint16_t *dhi,
                                                           const uint8_t *proto, const int *cls_proto,
                                                           uint32_t *lines) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    for (int64_t li = gw; li < nlines; li += nw) {
        const MsLineDesc L = desc[li];
        const int pcl = L.d == MSD_SPORT ? __ldg(cls_proto + L.c) : -1;
        uint32_t mine = 0;
#pragma unroll 4
        for (int k = 0; k < 32; k++) {
            const int64_t r = (int64_t)L.b * 1024 + k * 32 + lane;
            bool m = false;
            if (r < n) {
                switch (L.d) {
                    case MSD_SRC: m = (L.v & __ldg(sm + r)) == __ldg(sb + r); break;   // model.py:119-121
                    case MSD_DST: m = (L.v & __ldg(dm + r)) == __ldg(db + r); break;
                    case MSD_SPORT: {                                                // model.py:144-145, 224-225
                        const int rp = __ldg(proto + r);
                        m = (uint32_t)__ldg(slo + r) <= L.v && L.v <= (uint32_t)__ldg(shi + r) &&
                            (rp == 0 || rp == pcl);
                        break;
                    }
                    default: m = (uint32_t)__ldg(dlo + r) <= L.v && L.v <= (uint32_t)__ldg(dhi + r); break;
                }
            }
            const uint32_t b = __ballot_sync(0xFFFFFFFFu, m);
            if (lane == k) mine = b;
        }
        lines[li * 32 + lane] = mine;
    }
}

// thread per (row, block) of one dimension: the row's block-local interval
// (the last block boundary <= the row's first value) -> its line index
__global__ void ms_ptr_kernel(const uint32_t *vals, int64_t rows, int64_t ivl, int is_sport, int64_t nblk,
                              const uint32_t *bnd, const uint32_t *boff, uint16_t *ptr, int64_t pstride) {
    const int64_t total = rows * nblk;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / nblk, b = t - row * nblk;
        const int64_t c = is_sport ? row / ivl : 0;
        const uint32_t v = __ldg(vals + (is_sport ? row - c * ivl : row));
        const uint32_t b0 = __ldg(boff + b), cnt = __ldg(boff + b + 1) - b0;
        uint32_t lo = 0, hi = cnt;  // first boundary > v
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(bnd + b0 + mid) <= v) lo = mid + 1;
            else hi = mid;
        }
        PFW_CHECK(lo >= 1 && c * cnt + lo - 1 < 65536);
        ptr[row * pstride + b] = (uint16_t)(c * cnt + lo - 1);
    }
}

// Summary rows from compressed rows: lane k of word j looks at block 32j+k's
// line of the row and tests it for a set bit.
__global__ void __launch_bounds__(MS_BLOCK) ms_sum_cmp_kernel(const uint32_t *lines, const uint32_t *loff,
                                                              const uint16_t *ptr, int64_t pstride, int64_t rows,
                                                              int64_t blocks, int64_t sw, uint32_t *sum) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    for (int64_t t = gw; t < rows * sw; t += nw) {
        const int64_t row = t / sw, j = t - row * sw, blk = j * 32 + lane;
        uint32_t any = 0;
        if (blk < blocks) {
            const uint4 *q = reinterpret_cast<const uint4 *>(
                lines + ((size_t)__ldg(loff + blk) + __ldg(ptr + row * pstride + blk)) * 32);
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint4 v = __ldg(q + k);
                any |= v.x | v.y | v.z | v.w;
            }
        }
        const uint32_t b = __ballot_sync(0xFFFFFFFFu, any != 0u);
        if (lane == 0) sum[row * sw + j] = b;
    }
}

struct MsView {
    const uint32_t *bits0;    // the four dimensions' rows, one allocation
    uint32_t off[4];          // word offset of each dimension's rows from bits0
    const uint32_t *ipb[2];   // src / dst boundaries
    const uint4 *ipc[2];      // per /16 block: first boundary index | count << 24, the first 6 boundaries' low halves
    const uint16_t *port[2];  // sport / dport -> interval
    const uint32_t *pbk[2];   // sport / dport buckets of 32 ports: 2048 boundary-bit words, 2048 u16 bases
    const uint8_t *cls;       // protocol -> class
    int64_t wp;
    uint32_t sp_rows;
#ifdef PFW_CHECKS
    uint32_t nrows[4];        // rows per dimension
    uint64_t words;           // words of the bits0 allocation
#endif
};

// Block summaries (SUM variant only; the other variants take the empty type)
struct MsSum {
    const uint32_t *sum[4];   // summary rows: bit k = block k of the row non-zero
    uint32_t sw;              // summary words per row
};
struct MsNoSum {};
// Compressed rows (CMP variant; also carries the summaries)
struct MsCmp {
    const uint32_t *sum[4];
    uint32_t sw;
    uint32_t pstride, nblk;   // u16 line indices per row, blocks per row
    const uint16_t *ptr;      // line indices of every dimension's rows
    uint64_t ptr_off[4];
    const uint32_t *lines;    // distinct lines, 32 words each
    const uint32_t *loff;     // [4 * nblk]: first line of (dimension, block)
    const uint16_t *head;     // rows x 8: the first 8 blocks' line indices, dense
    uint64_t head_off[4];
};
template <bool SUM, bool CMP>
struct MsArg {
    using type = std::conditional_t<CMP, MsCmp, std::conditional_t<SUM, MsSum, MsNoSum>>;
};

// interval of an IP: index of the last boundary <= ip (boundary 0 is 0).
// c[ip >> 16] (16 bytes, one sector) packs the /16 block's first boundary
// index (24 bits), its boundary count (8 bits; 255: up to the next block's
// first) and the low 16 bits of its first 6 boundaries (0xFFFF past the
// count): blocks with <= 6 boundaries -- nearly all -- resolve from that one
// load (count of in-block boundaries <= ip), denser blocks binary-search b.
__device__ __forceinline__ uint32_t ms_ip_row(const uint32_t *b, const uint4 *c, uint32_t ip) {
    const uint4 e = __ldg(c + (ip >> 16));
    const uint32_t first = e.x & 0xFFFFFFu, cnt = e.x >> 24;
    if (cnt <= 6u) {
        const uint32_t l = ip & 0xFFFFu;
        uint32_t le = 0;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const uint32_t h = k == 0 ? e.y : k == 1 ? e.z : e.w;
            le += ((h & 0xFFFFu) <= l) + ((h >> 16) <= l);
        }
        // (the 0xFFFF padding counts only for ip low half 0xFFFF: take it back)
        return first - 1u + le - (l == 0xFFFFu ? 6u - cnt : 0u);
    }
    uint32_t lo = first;
    uint32_t hi = cnt == 255u ? (__ldg(&c[(ip >> 16) + 1].x) & 0xFFFFFFu) : lo + cnt;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(b + mid) <= ip) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

// port -> interval from the 32-port bucket table (two independent L1-resident
// loads; the lean plain-row kernel, whose carveout leaves L1 room for them --
// the compressed-row / summary kernels' larger shared memory does not: -1%)
__device__ __forceinline__ uint32_t ms_port_row(const uint32_t *bk, uint32_t port) {
    const uint32_t b = port >> 5;
    const uint32_t base = __ldg(reinterpret_cast<const uint16_t *>(bk + 2048) + b);
    return base + (uint32_t)__popc(__ldg(bk + b) & (0xFFFFFFFFu >> (31u - (port & 31u))));
}

// The four rows' words of one step, loaded by one asm block so that all four
// loads are in flight together (ptxas otherwise may hold the last one back
// behind the first three to save registers: two L2 round trips per step).
template <int V>
struct MsStep;
template <>
struct MsStep<4> {
    uint32_t w[4][4];
    __device__ __forceinline__ void load(const uint32_t *a, const uint32_t *b, const uint32_t *c,
                                         const uint32_t *d) {
        asm volatile(
            "ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%16];\n\t"
            "ld.global.nc.v4.u32 {%4, %5, %6, %7}, [%17];\n\t"
            "ld.global.nc.v4.u32 {%8, %9, %10, %11}, [%18];\n\t"
            "ld.global.nc.v4.u32 {%12, %13, %14, %15}, [%19];"
            : "=r"(w[0][0]), "=r"(w[0][1]), "=r"(w[0][2]), "=r"(w[0][3]), "=r"(w[1][0]), "=r"(w[1][1]),
              "=r"(w[1][2]), "=r"(w[1][3]), "=r"(w[2][0]), "=r"(w[2][1]), "=r"(w[2][2]), "=r"(w[2][3]),
              "=r"(w[3][0]), "=r"(w[3][1]), "=r"(w[3][2]), "=r"(w[3][3])
            : "l"(a), "l"(b), "l"(c), "l"(d));
    }
};
template <>
struct MsStep<2> {
    uint32_t w[4][2];
    __device__ __forceinline__ void load(const uint32_t *a, const uint32_t *b, const uint32_t *c,
                                         const uint32_t *d) {
        asm volatile(
            "ld.global.nc.v2.u32 {%0, %1}, [%8];\n\t"
            "ld.global.nc.v2.u32 {%2, %3}, [%9];\n\t"
            "ld.global.nc.v2.u32 {%4, %5}, [%10];\n\t"
            "ld.global.nc.v2.u32 {%6, %7}, [%11];"
            : "=r"(w[0][0]), "=r"(w[0][1]), "=r"(w[1][0]), "=r"(w[1][1]), "=r"(w[2][0]), "=r"(w[2][1]),
              "=r"(w[3][0]), "=r"(w[3][1])
            : "l"(a), "l"(b), "l"(c), "l"(d));
    }
};
template <>
struct MsStep<1> {
    uint32_t w[4][1];
    __device__ __forceinline__ void load(const uint32_t *a, const uint32_t *b, const uint32_t *c,
                                         const uint32_t *d) {
        asm volatile(
            "ld.global.nc.u32 %0, [%4];\n\t"
            "ld.global.nc.u32 %1, [%5];\n\t"
            "ld.global.nc.u32 %2, [%6];\n\t"
            "ld.global.nc.u32 %3, [%7];"
            : "=r"(w[0][0]), "=r"(w[1][0]), "=r"(w[2][0]), "=r"(w[3][0])
            : "l"(a), "l"(b), "l"(c), "l"(d));
    }
};

// Warps own batches of 32 packets (grid-stride).  Lane l looks up packet l's
// four rows (word offsets into shared memory).  The warp then works as 32/G
// independent groups of G lanes: each group searches one packet, reading V
// consecutive words per lane of each of the packet's four rows per step
// (G*V words = 32*G*V rules, one vector load per row per lane), ANDs them;
// one ballot per iteration serves every group (the group's slice of it finds
// its first non-zero word).  A group that finishes its packet (match, or
// window exhausted) takes the batch's next packet at once, so groups advance
// independently and the warp's loads stay spread over 32/G packets.
// WIN: the window is not the whole table, so the first / last step mask
// words outside it (a whole-table scan needs no masks: bits past the last
// rule are zero and rows are whole steps long).
// SUM (G*V = 32 words: one step = one 1024-rule block): with the first step
// a group also loads the packet's four summary rows (bit k = block k of the
// row has a bit set; lane gl holds blocks 32*gl..32*gl+31) and ANDs them;
// later steps jump to the next block whose AND-summary bit is set, skipping
// blocks no rule of which can match this packet (a set bit may still be a
// false candidate: the block is then read and the search moves on).
// CMP: the rows are compressed (MatchSet::cmp): the lookup phase also parks
// each packet's absolute line numbers (loff[d][block] + index) for 8 blocks
// in shared memory; a step reads those lines (beyond the 8 blocks the index
// comes from global memory).
template <int MODE, int G, int V, bool WIN, bool SUM = false, bool CMP = false>
__global__ void __launch_bounds__(MS_BLOCK, (SUM && CMP) ? PFW_MS_MINB_SC : PFW_MS_MINB)
    ms_scan_kernel(ScanParams p, MsView t, typename MsArg<SUM, CMP>::type u) {
    static_assert(!(SUM || CMP) || G * V == 32, "summary / compressed blocks are one step");
    constexpr int P = 32 / G;                      // packets in flight per warp
    constexpr uint32_t STEP = (uint32_t)G * V;     // words per step
    constexpr uint32_t GMASK = G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u);
    constexpr int LPB = PFW_MS_LPB, BATCH = 32 * LPB;  // packets per warp batch
    __shared__ uint4 s_off[CMP ? 1 : MS_BLOCK / 32][CMP ? 1 : BATCH];  // per warp: row offsets (plain rows)
    __shared__ uint4 s_row[(SUM || CMP) ? MS_BLOCK / 32 : 1][BATCH];  // per warp: row indices (SUM / CMP)
    __shared__ uint32_t s_lnum[CMP ? MS_BLOCK / 32 : 1][CMP ? BATCH : 1][4 * PFW_MS_PARK];
    // SUM && CMP: each packet's first PFW_MS_PARK candidate blocks (AND-summary
    // bits) -- their block numbers here, their line numbers in s_lnum -- and
    // the count (bit 7: more candidates follow the parked ones)
    __shared__ uint16_t s_cb[(SUM && CMP) ? MS_BLOCK / 32 : 1][(SUM && CMP) ? BATCH : 1][PFW_MS_PARK];
    __shared__ uint8_t s_nc[(SUM && CMP) ? MS_BLOCK / 32 : 1][(SUM && CMP) ? BATCH : 1];  // CMP: line numbers, 8 blocks x 4 dims (u32)
    __shared__ uint32_t s_res[MS_BLOCK / 32][BATCH];  // per warp: first match (word base until resolved)
    __shared__ uint32_t s_xw[MS_BLOCK / 32][BATCH][V];  // per packet: the finding lane's AND words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / G, gl = lane % G, gbase = grp * G;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t n = p.n;
    const uint32_t span = (uint32_t)(p.win_hi > p.win_lo ? p.win_hi - p.win_lo : 0);
    const bool empty = p.lo >= p.hi;
    const uint32_t wlo = (uint32_t)(p.lo >> 5), whi = empty ? 0u : (uint32_t)((p.hi - 1) >> 5);
    const uint32_t cbeg = wlo & ~(STEP - 1u);      // step-aligned start
    const int nsteps = empty ? 0 : (int)((whi - cbeg) / STEP) + 1;
    // this lane's masks on the first and the last step (WIN)
    uint32_t mfirst[V], mlast[V];
#pragma unroll
    for (int v = 0; v < V; v++) {
        const uint32_t w0 = cbeg + (uint32_t)gl * V + v;
        const uint32_t wl = cbeg + (uint32_t)(nsteps - 1) * STEP + (uint32_t)gl * V + v;
        mfirst[v] = w0 < wlo ? 0u : (w0 == wlo ? (0xFFFFFFFFu << (p.lo & 31)) : 0xFFFFFFFFu);
        mlast[v] = wl > whi ? 0u : (wl == whi ? (0xFFFFFFFFu >> (31 - ((p.hi - 1) & 31))) : 0xFFFFFFFFu);
    }
    const uint32_t lv = (uint32_t)gl * V;
    const uint32_t cab = (cbeg / 32u) & ~7u;  // CMP: first block of the parked line indices
    unsigned long long st_sum = 0, st_blocks = 0;
    unsigned st_max = 0;

    for (int64_t b0 = gw * BATCH; b0 < n; b0 += nw * BATCH) {
        const int nv = (int)((n - b0) < BATCH ? (n - b0) : BATCH);
        // the batch's packets (all LPB loads in flight), then their rows
        uint4 v[LPB];
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            v[k] = make_uint4(0u, 0u, 0u, 0u);
            if (i < n) {
                if (p.pkts) {
                    v[k] = __ldcs(p.pkts + i);  // streamed once: evict-first in L2 (the tables stay)
                } else {
                    v[k].x = __ldcs(p.cols.src + i);
                    v[k].y = __ldcs(p.cols.dst + i);
                    v[k].z = ((uint32_t)__ldcs(p.cols.sport + i) << 16) | (uint32_t)__ldcs(p.cols.dport + i);
                    v[k].w = __ldcs(p.cols.proto + i);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            if (i < n) {
                const uint32_t wp = (uint32_t)t.wp;
                const uint4 r = make_uint4(
                    ms_ip_row(t.ipb[0], t.ipc[0], v[k].x), ms_ip_row(t.ipb[1], t.ipc[1], v[k].y),
                    (uint32_t)__ldg(t.cls + (v[k].w & 0xFFu)) * t.sp_rows + __ldg(t.port[0] + (v[k].z >> 16)),
                    __ldg(t.port[1] + (v[k].z & 0xFFFFu)));
                PFW_CHECK(r.x < t.nrows[0] && r.y < t.nrows[1] && r.z < t.nrows[2] && r.w < t.nrows[3]);
                // word offsets from the common base, at the first step
                if (!CMP)
                    s_off[CMP ? 0 : warp][CMP ? 0 : k * 32 + lane] =
                        make_uint4(r.x * wp + cbeg + t.off[0], r.y * wp + cbeg + t.off[1], r.z * wp + cbeg + t.off[2],
                                   r.w * wp + cbeg + t.off[3]);
                if (SUM || CMP) s_row[(SUM || CMP) ? warp : 0][k * 32 + lane] = r;
                if constexpr (SUM && CMP) {
                    // lane-parallel (one packet per lane): the packet's candidate
                    // blocks in [blk0, blast] -- set bits of the AND of its four
                    // summary rows -- and the line numbers of the first
                    // PFW_MS_PARK of them, so the group loop just walks the list
                    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
                    const uint32_t kb0 = cbeg / 32u, kb1 = whi / 32u;
                    uint32_t *dst = &s_lnum[CMP ? warp : 0][CMP ? k * 32 + lane : 0][0];
                    uint16_t *cbl = &s_cb[(SUM && CMP) ? warp : 0][(SUM && CMP) ? k * 32 + lane : 0][0];
                    int nc = 0, more = 0;
                    for (uint32_t w = kb0 / 32u; w <= kb1 / 32u && !more; w++) {
                        uint32_t a = __ldg(u.sum[0] + (size_t)r.x * u.sw + w) & __ldg(u.sum[1] + (size_t)r.y * u.sw + w) &
                                     __ldg(u.sum[2] + (size_t)r.z * u.sw + w) & __ldg(u.sum[3] + (size_t)r.w * u.sw + w);
                        const int rel0 = (int)kb0 - 32 * (int)w, rel1 = (int)kb1 - 32 * (int)w;
                        a &= rel0 <= 0 ? 0xFFFFFFFFu : (rel0 >= 32 ? 0u : (0xFFFFFFFFu << rel0));
                        a &= rel1 < 0 ? 0u : (rel1 >= 31 ? 0xFFFFFFFFu : ((2u << rel1) - 1u));
                        while (a) {
                            if (nc == PFW_MS_PARK) {
                                more = 1;
                                break;
                            }
                            const uint32_t b = 32u * w + (uint32_t)(__ffs(a) - 1);
                            a &= a - 1u;
                            cbl[nc] = (uint16_t)b;
#pragma unroll
                            for (int d = 0; d < 4; d++) {
                                const uint16_t ix = b < 8u ? __ldg(u.head + u.head_off[d] + (size_t)rr[d] * 8 + b)
                                                           : __ldg(u.ptr + u.ptr_off[d] + (size_t)rr[d] * u.pstride + b);
                                dst[PFW_MS_PARK * d + nc] = __ldg(u.loff + d * u.nblk + b) + ix;
                            }
                            nc++;
                        }
                    }
                    s_nc[(SUM && CMP) ? warp : 0][(SUM && CMP) ? k * 32 + lane : 0] = (uint8_t)(nc | (more << 7));
                } else if constexpr (CMP) {
                    // absolute line numbers (loff + index) of the 8 blocks from
                    // the 8-aligned block at or below the first, per dimension
                    const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        // (whole-table scans start at block 0: the dense head array)
                        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(
                            cab == 0 ? u.head + u.head_off[d] + (size_t)rr[d] * 8
                                     : u.ptr + u.ptr_off[d] + (size_t)rr[d] * u.pstride + cab));
                        const uint32_t *lo = u.loff + d * u.nblk + cab;  // (loff has 8 entries of slack)
                        const uint32_t qq[4] = {q.x, q.y, q.z, q.w};
                        uint32_t *dst = &s_lnum[CMP ? warp : 0][CMP ? k * 32 + lane : 0][PFW_MS_PARK * d];
#pragma unroll
                        for (int jj = 0; jj < PFW_MS_PARK; jj++)
                            dst[jj] = __ldg(lo + jj) + ((qq[jj >> 1] >> (16 * (jj & 1))) & 0xFFFFu);
                    }
                }
            }
            s_res[warp][k * 32 + lane] = PFW_NO_MATCH;
        }
        __syncwarp();
        if (nsteps > 0) {
            // group state (group-uniform): packet pj (-1 idle), step s, the
            // packet's four row offsets at this lane's words of step s.
            // Packets are handed out in group order, so once every packet is
            // taken the idle-group count is next - nv: the loop ends when it
            // reaches P.
            int pj = grp < nv ? grp : -1;
            int next = P;
            int s = 0;
            uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
            uint32_t scand = 0;  // SUM: candidate blocks after the current one (this lane's 32)
            unsigned nrd = 0;    // SUM: block reads of this lane's group (counted on lane gl == 0)
            int ck = 0;          // SUM && CMP: index into the packet's parked candidate list
            bool fb = false;     // SUM && CMP: past the parked candidates (in-loop summary search)
            bool fbload = false; // SUM && CMP: load the summaries this iteration (switching to fb)
            const uint32_t blk0 = cbeg / 32u, blast = whi / 32u;  // SUM: first / last block
            if (pj >= 0) {
                const uint4 o = s_off[CMP ? 0 : warp][CMP ? 0 : pj];
                o0 = o.x + lv;
                o1 = o.y + lv;
                o2 = o.z + lv;
                o3 = o.w + lv;
            }
            while (next < nv + P) {
                const bool act = pj >= 0;
                uint32_t x[V], any = 0u;
#pragma unroll
                for (int v = 0; v < V; v++) x[v] = 0u;
                if constexpr (SUM && CMP) {
                    if (act && fbload) {
                        // past the parked candidates: the AND-summary after the last one
                        scand = 0u;
                        if ((uint32_t)gl < u.sw) {
                            const uint4 rw = s_row[(SUM || CMP) ? warp : 0][pj];
                            scand = __ldg(u.sum[0] + (size_t)rw.x * u.sw + gl) &
                                    __ldg(u.sum[1] + (size_t)rw.y * u.sw + gl) &
                                    __ldg(u.sum[2] + (size_t)rw.z * u.sw + gl) &
                                    __ldg(u.sum[3] + (size_t)rw.w * u.sw + gl);
                            const int rel0 = (int)(blk0 + (uint32_t)s) - 32 * gl, rel1 = (int)blast - 32 * gl;
                            scand &= rel0 < 0 ? 0xFFFFFFFFu : (rel0 >= 31 ? 0u : (0xFFFFFFFFu << (rel0 + 1)));
                            scand &= rel1 < 0 ? 0u : (rel1 >= 31 ? 0xFFFFFFFFu : ((2u << rel1) - 1u));
                        }
                    }
                } else if constexpr (SUM) {
                    if (act && s == 0) {
                        // the packet's first step: its AND-summary, restricted
                        // to the blocks after this one, up to the window's last
                        scand = 0u;
                        if ((uint32_t)gl < u.sw) {
                            const uint4 rw = s_row[(SUM || CMP) ? warp : 0][pj];
                            PFW_CHECK(rw.x < t.nrows[0] && rw.y < t.nrows[1] && rw.z < t.nrows[2] && rw.w < t.nrows[3]);
                            scand = __ldg(u.sum[0] + (size_t)rw.x * u.sw + gl) &
                                    __ldg(u.sum[1] + (size_t)rw.y * u.sw + gl) &
                                    __ldg(u.sum[2] + (size_t)rw.z * u.sw + gl) &
                                    __ldg(u.sum[3] + (size_t)rw.w * u.sw + gl);
                            const int rel0 = (int)blk0 - 32 * gl, rel1 = (int)blast - 32 * gl;
                            scand &= rel0 < 0 ? 0xFFFFFFFFu : (rel0 >= 31 ? 0u : (0xFFFFFFFFu << (rel0 + 1)));
                            scand &= rel1 < 0 ? 0u : (rel1 >= 31 ? 0xFFFFFFFFu : ((2u << rel1) - 1u));
                        }
                    }
                }
                // this iteration reads lines (SUM && CMP: a parked candidate, or a
                // fallback step; not the summary-only switching iteration)
                const int pnc = (SUM && CMP && act) ? (int)s_nc[(SUM && CMP) ? warp : 0][(SUM && CMP) ? pj : 0] : 0;
                const bool rd = act && (!(SUM && CMP) || (fb ? !fbload : ck < (pnc & 0x7F)));
                if (SUM && rd && gl == 0) nrd++;
                PFW_CHECK(!act || (pj < nv && (CMP || (uint64_t)max(max(o0, o1), max(o2, o3)) + V <= t.words)));
                uint32_t x2[V], any2 = 0u;  // SUM && CMP list walk: the second candidate of this step
                bool two = false;
                int s2 = 0;
#pragma unroll
                for (int v = 0; v < V; v++) x2[v] = 0u;
                if (rd) {
                    MsStep<V> st;
                    if constexpr (SUM && CMP) {
                        uint32_t q0, q1, q2, q3, b;
                        if (!fb) {  // the next parked candidate(s): two per step when there are
                            b = s_cb[(SUM && CMP) ? warp : 0][(SUM && CMP) ? pj : 0][ck];
                            const uint32_t *sp = &s_lnum[CMP ? warp : 0][CMP ? pj : 0][0];
                            q0 = sp[ck];
                            q1 = sp[PFW_MS_PARK + ck];
                            q2 = sp[2 * PFW_MS_PARK + ck];
                            q3 = sp[3 * PFW_MS_PARK + ck];
                            s = (int)(b - blk0);
                            two = ck + 1 < (pnc & 0x7F);
                            if (two) {
                                if (gl == 0) nrd++;  // (a second block read this step)
                                const uint32_t b2 = s_cb[(SUM && CMP) ? warp : 0][(SUM && CMP) ? pj : 0][ck + 1];
                                s2 = (int)(b2 - blk0);
                                MsStep<V> st2;
                                const uint32_t *l2 = u.lines + lv;
                                st2.load(l2 + ((size_t)sp[ck + 1] << 5), l2 + ((size_t)sp[PFW_MS_PARK + ck + 1] << 5),
                                         l2 + ((size_t)sp[2 * PFW_MS_PARK + ck + 1] << 5),
                                         l2 + ((size_t)sp[3 * PFW_MS_PARK + ck + 1] << 5));
#pragma unroll
                                for (int v = 0; v < V; v++) {
                                    x2[v] = st2.w[0][v] & st2.w[1][v] & st2.w[2][v] & st2.w[3][v];
                                    if (WIN) {
                                        if (s2 == 0) x2[v] &= mfirst[v];
                                        if (s2 == nsteps - 1) x2[v] &= mlast[v];
                                    }
                                    any2 |= x2[v];
                                }
                            }
                        } else {    // in-loop summary search: line numbers from global memory
                            b = blk0 + (uint32_t)s;
                            const uint4 rw = s_row[(SUM || CMP) ? warp : 0][pj];
                            q0 = __ldg(u.loff + b) + __ldg(u.ptr + u.ptr_off[0] + (size_t)rw.x * u.pstride + b);
                            q1 = __ldg(u.loff + u.nblk + b) + __ldg(u.ptr + u.ptr_off[1] + (size_t)rw.y * u.pstride + b);
                            q2 = __ldg(u.loff + 2 * u.nblk + b) + __ldg(u.ptr + u.ptr_off[2] + (size_t)rw.z * u.pstride + b);
                            q3 = __ldg(u.loff + 3 * u.nblk + b) + __ldg(u.ptr + u.ptr_off[3] + (size_t)rw.w * u.pstride + b);
                        }
                        PFW_CHECK(b >= blk0 && b <= blast);
                        const uint32_t *l = u.lines + lv;
                        st.load(l + ((size_t)q0 << 5), l + ((size_t)q1 << 5), l + ((size_t)q2 << 5),
                                l + ((size_t)q3 << 5));
                    } else if constexpr (CMP) {
                        const uint32_t b = cbeg / 32u + (uint32_t)s;  // this step's block
                        const int j = (int)(b - cab);
                        uint32_t q0, q1, q2, q3;  // absolute line numbers
                        if (j < PFW_MS_PARK) {
                            const uint32_t *sp = &s_lnum[CMP ? warp : 0][CMP ? pj : 0][0];
                            q0 = sp[j];
                            q1 = sp[PFW_MS_PARK + j];
                            q2 = sp[2 * PFW_MS_PARK + j];
                            q3 = sp[3 * PFW_MS_PARK + j];
                        } else {
                            const uint4 rw = s_row[(SUM || CMP) ? warp : 0][pj];
                            q0 = __ldg(u.loff + b) + __ldg(u.ptr + u.ptr_off[0] + (size_t)rw.x * u.pstride + b);
                            q1 = __ldg(u.loff + u.nblk + b) + __ldg(u.ptr + u.ptr_off[1] + (size_t)rw.y * u.pstride + b);
                            q2 = __ldg(u.loff + 2 * u.nblk + b) + __ldg(u.ptr + u.ptr_off[2] + (size_t)rw.z * u.pstride + b);
                            q3 = __ldg(u.loff + 3 * u.nblk + b) + __ldg(u.ptr + u.ptr_off[3] + (size_t)rw.w * u.pstride + b);
                        }
                        const uint32_t *l = u.lines + lv;
                        st.load(l + ((size_t)q0 << 5), l + ((size_t)q1 << 5), l + ((size_t)q2 << 5),
                                l + ((size_t)q3 << 5));
                    } else {
                        st.load(t.bits0 + o0, t.bits0 + o1, t.bits0 + o2, t.bits0 + o3);
                    }
#pragma unroll
                    for (int v = 0; v < V; v++) {
                        x[v] = st.w[0][v] & st.w[1][v] & st.w[2][v] & st.w[3][v];
                        if (WIN) {
                            if (s == 0) x[v] &= mfirst[v];
                            if (s == nsteps - 1) x[v] &= mlast[v];
                        }
                        any |= x[v];
                    }
                }
                unsigned bal = __ballot_sync(0xFFFFFFFFu, any != 0u);
                uint32_t gbits = (bal >> gbase) & GMASK;
                if constexpr (SUM && CMP) {
                    // a group whose first candidate of the step has no match takes
                    // the second one's (its blocks are later: still the lowest)
                    const unsigned bal2 = __ballot_sync(0xFFFFFFFFu, any2 != 0u && gbits == 0u);
                    const uint32_t gbits2 = (bal2 >> gbase) & GMASK;
                    if (gbits2) {
                        gbits = gbits2;
                        s = s2;
#pragma unroll
                        for (int v = 0; v < V; v++) x[v] = x2[v];
                    }
                    bal |= bal2;
                    if (two && !gbits2 && gbits == 0u) s = s2;  // (the last block this step read)
                }
                const bool found = gbits != 0u;  // (idle groups have no bits)
                if (found) {
                    // the group's lowest lane with a set bit parks its words and
                    // their position; the bit is resolved after the loop, one
                    // packet per lane
                    uint32_t anyx = 0u;
#pragma unroll
                    for (int v = 0; v < V; v++) anyx |= x[v];
                    if (anyx != 0u && (gbits & ((1u << gl) - 1u)) == 0u) {
                        s_res[warp][pj] = cbeg + (uint32_t)s * STEP + lv;
#pragma unroll
                        for (int v = 0; v < V; v++) s_xw[warp][pj][v] = x[v];
                    }
                }
                bool done = act && (found || s + 1 >= nsteps);
                int ns = s + 1;  // next step (SUM: the next candidate block)
                bool sw_fb = false;  // SUM && CMP: switch to the in-loop summary search
                if constexpr (SUM && CMP) {
                    if (!fb) {
                        // walking the parked list: done, next parked, or switch
                        const int nc = pnc & 0x7F, more = pnc >> 7, nxt = ck + (two ? 2 : 1);
                        done = act && (found || (nxt >= nc && !more));
                        sw_fb = act && !done && nxt >= nc;  // (more candidates after the parked ones)
                    }
                }
                // (SUM && CMP: only while some group of the warp is past its parked candidates)
                if (SUM && (!CMP || __any_sync(0xFFFFFFFFu, fb))) {
                    // next candidate block of the groups still searching
                    const bool fbs = !CMP || fb;  // groups in the in-loop summary search
                    const uint32_t cm = (act && !found && fbs) ? scand : 0u;
                    const uint32_t cbits = (__ballot_sync(0xFFFFFFFFu, cm != 0u) >> gbase) & GMASK;
                    const int nb = __shfl_sync(0xFFFFFFFFu, 32 * gl + __ffs(cm) - 1,
                                               gbase + (__ffs(cbits) - 1) * (cbits != 0u));
                    if (fbs) done = act && (found || cbits == 0u);
                    if (fbs && !done && act) {
                        ns = nb - (int)blk0;
                        const int rel = nb - 32 * gl;  // drop candidates up to nb
                        scand &= rel < 0 ? 0xFFFFFFFFu : (rel >= 31 ? 0u : (0xFFFFFFFFu << (rel + 1)));
                    }
                }
                const unsigned dmask = __ballot_sync(0xFFFFFFFFu, done && gl == 0);
                if (done) {
                    // take the next packet (rank of this group among the done ones)
                    const int np = next + __popc(dmask & ((1u << gbase) - 1u));
                    pj = np < nv ? np : -1;
                    s = 0;
                    ck = 0;
                    fb = false;
                    fbload = false;
                    if (pj >= 0) {
                        const uint4 o = s_off[CMP ? 0 : warp][CMP ? 0 : pj];
                        o0 = o.x + lv;
                        o1 = o.y + lv;
                        o2 = o.z + lv;
                        o3 = o.w + lv;
                    }
                } else if (act) {
                    if constexpr (SUM && CMP) {
                        if (!fb) {
                            if (sw_fb) {
                                fb = true;      // next iteration: load the summaries after block blk0 + s
                                fbload = true;
                            } else {
                                ck += two ? 2 : 1;
                            }
                        } else {
                            fbload = false;
                            s = ns;
                        }
                    } else if constexpr (SUM) {
                        const uint32_t adv = (uint32_t)(ns - s) * STEP;
                        s = ns;
                        o0 += adv;
                        o1 += adv;
                        o2 += adv;
                        o3 += adv;
                    } else {
                        s++;
                        o0 += STEP;
                        o1 += STEP;
                        o2 += STEP;
                        o3 += STEP;
                    }
                }
                next += __popc(dmask);
            }
            if constexpr (SUM) st_blocks += nrd;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            if (i < n) {
                uint32_t res = s_res[warp][k * 32 + lane];
                if (res != PFW_NO_MATCH) {  // the parked words' first non-zero word, its lowest bit
                    const uint32_t *xw = s_xw[warp][k * 32 + lane];
                    uint32_t wsel = xw[V - 1], widx = V - 1;
#pragma unroll
                    for (int v = V - 2; v >= 0; v--) {
                        const uint32_t xv = xw[v];
                        wsel = xv ? xv : wsel;
                        widx = xv ? (uint32_t)v : widx;
                    }
                    res = (res + widx) * 32u + (uint32_t)(__ffs(wsel) - 1);
                }
                PFW_CHECK(res == PFW_NO_MATCH || (res >= p.lo && res < p.hi));
                emit_result<MODE, true>(p, (uint32_t)i, res, span, st_sum, st_max);
            }
        }
        __syncwarp();
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
    if constexpr (SUM) {
        if (p.blocks_read) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) st_blocks += __shfl_xor_sync(0xFFFFFFFFu, st_blocks, o);
            if (lane == 0 && st_blocks) atomicAdd(p.blocks_read, st_blocks);
        }
    }
}

// base + 4 * off as one IMAD.WIDE (base: a 64-bit per-lane register)
__device__ __forceinline__ const uint32_t *ms_word_ptr(const uint32_t *base, uint32_t off) {
    const uint32_t *r;
    asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(r) : "r"(off), "l"(base));
    return r;
}

// The four rows' V words of one step for this lane: 128-bit loads (V = 4)
// or Blackwell's 256-bit loads (V = 8, LDG.E.ENL2.256), all four in flight
// together.
template <int V>
__device__ __forceinline__ void ms_load_rows(const uint32_t *a, const uint32_t *b, const uint32_t *c,
                                             const uint32_t *d, uint32_t (&w)[4][V]) {
    if constexpr (V == 8) {
        asm volatile(
            "ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%32];\n\t"
            "ld.global.nc.v8.u32 {%8, %9, %10, %11, %12, %13, %14, %15}, [%33];\n\t"
            "ld.global.nc.v8.u32 {%16, %17, %18, %19, %20, %21, %22, %23}, [%34];\n\t"
            "ld.global.nc.v8.u32 {%24, %25, %26, %27, %28, %29, %30, %31}, [%35];"
            : "=r"(w[0][0]), "=r"(w[0][1]), "=r"(w[0][2]), "=r"(w[0][3]), "=r"(w[0][4]), "=r"(w[0][5]),
              "=r"(w[0][6]), "=r"(w[0][7]), "=r"(w[1][0]), "=r"(w[1][1]), "=r"(w[1][2]), "=r"(w[1][3]),
              "=r"(w[1][4]), "=r"(w[1][5]), "=r"(w[1][6]), "=r"(w[1][7]), "=r"(w[2][0]), "=r"(w[2][1]),
              "=r"(w[2][2]), "=r"(w[2][3]), "=r"(w[2][4]), "=r"(w[2][5]), "=r"(w[2][6]), "=r"(w[2][7]),
              "=r"(w[3][0]), "=r"(w[3][1]), "=r"(w[3][2]), "=r"(w[3][3]), "=r"(w[3][4]), "=r"(w[3][5]),
              "=r"(w[3][6]), "=r"(w[3][7])
            : "l"(a), "l"(b), "l"(c), "l"(d));
    } else {
        static_assert(V == 4, "4 or 8 words per lane");
        MsStep<4> st;
        st.load(a, b, c, d);
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int k = 0; k < 4; k++) w[r][k] = st.w[r][k];
    }
}

// The first set bit of a finding lane's parked AND words (V words starting at
// word index wbase of the row): (wbase + first non-zero word) * 32 + its lowest bit
template <int V>
__device__ __forceinline__ uint32_t ms_parked_first_bit(const uint4 *px, uint32_t wbase) {
    uint32_t x[V];
#pragma unroll
    for (int k = 0; k < V; k += 4) {
        const uint4 q4 = px[k / 4];
        x[k] = q4.x;
        x[k + 1] = q4.y;
        x[k + 2] = q4.z;
        x[k + 3] = q4.w;
    }
    uint32_t wsel = x[V - 1], widx = V - 1;
#pragma unroll
    for (int k = V - 2; k >= 0; k--) {
        wsel = x[k] ? x[k] : wsel;
        widx = x[k] ? (uint32_t)k : widx;
    }
    return (wbase + widx) * 32u + (uint32_t)(__ffs(wsel) - 1);
}

// Lean scan of whole-table windows over plain rows (the data-parallel /
// grid / sequential configs): the search of ms_scan_kernel<MODE, G, V,
// false> -- groups of G lanes, one 128-byte line of each of the packet's four
// rows per step (1024 rules), groups refilled from the warp's batch of 32 --
// with the per-step work cut to what the search needs:
//  * idle groups read a zero line (the padding after the src rows) instead
//    of being predicated off, so no per-iteration zeroing / predicate setup;
//  * the group's lowest lane with a set bit parks its AND words; the bit is
//    resolved after the loop, one packet per lane; the next state is
//    selected branch-free;
//  * G = 4: each lane loads 32 bytes per row (256-bit loads), so one load
//    instruction per row serves 8 packets per warp (8 steps per iteration).
// Results are identical (same lowest set bit of the same AND).
template <int MODE, int G, int V, int LPB, int MINB>
__global__ void __launch_bounds__(MS_BLOCK, MINB)
    ms_lean_kernel(ScanParams p, MsView t, uint32_t zoff) {
    constexpr int P = 32 / G;                   // packets in flight per warp
    constexpr int B = 32 * LPB;                 // packets per warp batch
    constexpr uint32_t STEP = (uint32_t)G * V;  // words per step (G*V = 32: one line per row)
    static_assert(V % 4 == 0 && 128 % STEP == 0, "4 or 8 words per lane; steps divide the 128-word row unit");
    __shared__ uint4 s_off[MS_BLOCK / 32][B + 1];  // per packet: its four rows' word offsets; [B]: the zero line
    __shared__ uint32_t s_res[MS_BLOCK / 32][B];   // per packet: word base of its first match (resolved after)
    __shared__ uint4 s_x[MS_BLOCK / 32][B][V / 4];  // per packet: the finding lane's AND words
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / G, gl = lane % G, gbase = grp * G;
    const uint32_t lv = (uint32_t)gl * V;
    const unsigned below = (1u << gl) - 1u;            // group lanes below this one (in group bits)
    const unsigned groups_below = (1u << gbase) - 1u;  // warp lanes of the groups below this one
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t n = p.n;
    const uint32_t span = (uint32_t)(p.win_hi > p.win_lo ? p.win_hi - p.win_lo : 0);
    const int nsteps = p.lo >= p.hi ? 0 : (int)((uint32_t)((p.hi - 1) >> 5) / STEP) + 1;
    const uint32_t wp = (uint32_t)t.wp;
    const uint32_t *bits = t.bits0;
    if (lane == 0) s_off[warp][B] = make_uint4(zoff, zoff, zoff, zoff);
    const uint32_t s_off_base = (uint32_t)__cvta_generic_to_shared(&s_off[warp][0]);
    unsigned long long st_sum = 0;
    unsigned st_max = 0;

    for (int64_t b0 = gw * B; b0 < n; b0 += nw * B) {
        const int nv = (int)((n - b0) < B ? (n - b0) : B);
        // lookups, one packet per lane per round (all LPB packet loads in flight first)
        uint4 v[LPB];
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            v[k] = make_uint4(0u, 0u, 0u, 0u);
            if (i < n) {
                if (p.pkts) {
                    v[k] = __ldcs(p.pkts + i);  // streamed once: evict-first in L2 (the tables stay)
                } else {
                    v[k].x = __ldcs(p.cols.src + i);
                    v[k].y = __ldcs(p.cols.dst + i);
                    v[k].z = ((uint32_t)__ldcs(p.cols.sport + i) << 16) | (uint32_t)__ldcs(p.cols.dport + i);
                    v[k].w = __ldcs(p.cols.proto + i);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            if (i < n) {
                const uint4 r = make_uint4(
                    ms_ip_row(t.ipb[0], t.ipc[0], v[k].x), ms_ip_row(t.ipb[1], t.ipc[1], v[k].y),
                    (uint32_t)__ldg(t.cls + (v[k].w & 0xFFu)) * t.sp_rows + ms_port_row(t.pbk[0], v[k].z >> 16),
                    ms_port_row(t.pbk[1], v[k].z & 0xFFFFu));
                PFW_CHECK(r.x < t.nrows[0] && r.y < t.nrows[1] && r.z < t.nrows[2] && r.w < t.nrows[3]);
                s_off[warp][k * 32 + lane] = make_uint4(r.x * wp + t.off[0], r.y * wp + t.off[1],
                                                        r.z * wp + t.off[2], r.w * wp + t.off[3]);
            }
            s_res[warp][k * 32 + lane] = PFW_NO_MATCH;
        }
        __syncwarp();
        if (nsteps > 0) {
            // group state: packet pj of the batch (-1: idle, reading the zero
            // line), step s, the four rows' word offsets at this lane's words
            // (s_off holds each packet's row offsets; a lane adds its own lv)
            int pj = grp < nv ? grp : -1;
            int next = P;  // next packet to hand out; every group idle <=> next == nv + P
            int s = 0;
            uint4 o = s_off[warp][pj >= 0 ? pj : B];
            o.x += lv;
            o.y += lv;
            o.z += lv;
            o.w += lv;
            while (next < nv + P) {
                PFW_CHECK((uint64_t)max(max(o.x, o.y), max(o.z, o.w)) + V <= t.words);
                uint32_t w[4][V];
                ms_load_rows<V>(bits + o.x, bits + o.y, bits + o.z, bits + o.w, w);
                uint32_t x[V], any = 0u;
#pragma unroll
                for (int k = 0; k < V; k++) {
                    x[k] = w[0][k] & w[1][k] & w[2][k] & w[3][k];
                    any |= x[k];
                }
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, any != 0u);
                const unsigned gbits = (bal >> gbase) & ((1u << G) - 1u);
                // the group's lowest lane with a set bit holds the packet's
                // first match: it parks its words and their position; the
                // bit itself is resolved after the loop, one packet per lane
                // (a 32-lane select chain instead of one per iteration)
                if (any != 0u && (gbits & below) == 0u) {
                    s_res[warp][pj] = (uint32_t)s * STEP + lv;  // word index of x[0]
#pragma unroll
                    for (int k = 0; k < V; k += 4) s_x[warp][pj][k / 4] = make_uint4(x[k], x[k + 1], x[k + 2], x[k + 3]);
                }
                const bool act = pj >= 0;
                const bool done = act && (gbits != 0u || s + 1 >= nsteps);
                const unsigned dm = __ballot_sync(0xFFFFFFFFu, done && gl == 0);
                // next state, branch-free: a finished group takes the batch's
                // next packet (its rank among the finished groups), an active
                // one advances one step, an idle one stays on the zero line
                const int np = next + __popc(dm & groups_below);
                const bool take = np < nv;
                // a finished group loads its next packet's offsets straight into
                // o (predicated shared load), then every lane adds lv (new
                // packet) or one step (active) or nothing (idle)
                {
                    const uint32_t sa = s_off_base + (uint32_t)(take ? np : B) * 16u;
                    asm volatile(
                        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
                        "@q ld.shared.v4.u32 {%0, %1, %2, %3}, [%5];\n\t}"
                        : "+r"(o.x), "+r"(o.y), "+r"(o.z), "+r"(o.w)
                        : "r"((uint32_t)done), "r"(sa)
                        : "memory");
                }
                const uint32_t add = done ? lv : (act ? STEP : 0u);
                o.x += add;
                o.y += add;
                o.z += add;
                o.w += add;
                s = done ? 0 : s + (act ? 1 : 0);
                pj = done ? (take ? np : -1) : pj;
                next += __popc(dm);
            }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < LPB; k++) {
            const int64_t i = b0 + k * 32 + lane;
            if (i < n) {
                uint32_t res = s_res[warp][k * 32 + lane];
                if (res != PFW_NO_MATCH) res = ms_parked_first_bit<V>(&s_x[warp][k * 32 + lane][0], res);
                PFW_CHECK(res == PFW_NO_MATCH || (res >= p.lo && res < p.hi));
                emit_result<MODE, true>(p, (uint32_t)i, res, span, st_sum, st_max);
            }
        }
        __syncwarp();
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

// Lean scan of whole-table windows over COMPRESSED rows (large rulesets, the
// function-parallel config): the lean kernel's step loop, where a step's four
// lines are line numbers instead of row offsets.  The lookup phase parks each
// packet's absolute line numbers (loff[d][b] + index) for its first MS_LEAN_PARK
// blocks in shared memory, from the dense head array (one 16-byte load per
// dimension); a step takes its block's four line numbers with one shared
// 16-byte load; a packet that walks past its parked window (rare: most scans
// end in the first two or three blocks) has its group park the next
// MS_LEAN_PARK blocks' line numbers, one block per lane.  Idle groups read the
// zero line after the last distinct line.
#ifndef MS_LEAN_PARK
#define MS_LEAN_PARK 6
#endif
#ifndef MS_CMP_MINB
#define MS_CMP_MINB PFW_MS_MINB
#endif
#ifndef MS_CP_BLOCKS
#define MS_CP_BLOCKS 256
#endif
template <int MODE, int G, bool CP = false>
__global__ void __launch_bounds__(MS_BLOCK, G == 4 ? 4 : MS_CMP_MINB)
    ms_lean_cmp_kernel(ScanParams p, MsView t, MsCmp u, uint32_t zline) {
    constexpr int V = 32 / G, P = 32 / G, K = MS_LEAN_PARK;
    static_assert(K >= 1 && K <= 8, "1..8 parked blocks (the head array holds 8)");
    // CP: a parked block is its four u16 line indices (8 bytes) and the
    // (dimension, block) line offsets sit in one shared table (<= MS_CP_BLOCKS
    // blocks); otherwise a parked block is its four absolute line numbers
    using Slot = std::conditional_t<CP, uint2, uint4>;
    __shared__ __align__(16) Slot s_ln[MS_BLOCK / 32][32][K];  // per packet: blocks of its parked window
    __shared__ uint4 s_lo[CP ? MS_CP_BLOCKS : 1];             // CP: loff of block b, x..w = dimension
    __shared__ uint4 s_row[MS_BLOCK / 32][32];    // per packet: its four rows (re-parking)
    __shared__ uint32_t s_res[MS_BLOCK / 32][32];
    // (a finished packet's line-number slots are reused for the finding lane's AND words)
    static_assert((CP ? V / 2 : V / 4) <= K, "the parked words fit the packet's line-number slots");
    static_assert(!CP || K % 2 == 0, "16-byte aligned parked words");
    if constexpr (CP) {
        for (int b = threadIdx.x; b < (int)u.nblk && b < MS_CP_BLOCKS; b += MS_BLOCK)
            s_lo[b] = make_uint4(__ldg(u.loff + b), __ldg(u.loff + u.nblk + b), __ldg(u.loff + 2 * u.nblk + b),
                                 __ldg(u.loff + 3 * u.nblk + b));
        __syncthreads();
    }
    // a slot's four line numbers for block b
    auto line4 = [&](const Slot &e, uint32_t b) -> uint4 {
        if constexpr (CP) {
            const uint4 lo = s_lo[b];
            return make_uint4(lo.x + (e.x & 0xFFFFu), lo.y + (e.x >> 16), lo.z + (e.y & 0xFFFFu), lo.w + (e.y >> 16));
        } else {
            return e;
        }
    };
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / G, gl = lane % G, gbase = grp * G;
    const uint32_t lv = (uint32_t)gl * V;
    const unsigned below = (1u << gl) - 1u;
    const unsigned groups_below = (1u << gbase) - 1u;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t n = p.n;
    const uint32_t span = (uint32_t)(p.win_hi > p.win_lo ? p.win_hi - p.win_lo : 0);
    const int nsteps = p.lo >= p.hi ? 0 : (int)((uint32_t)((p.hi - 1) >> 5) / 32u) + 1;  // blocks
    const uint32_t *lines = u.lines;
    const uint4 zq = make_uint4(zline, zline, zline, zline);
    unsigned long long st_sum = 0;
    unsigned st_max = 0;

    for (int64_t b0 = gw * 32; b0 < n; b0 += nw * 32) {
        const int nv = (int)((n - b0) < 32 ? (n - b0) : 32);
        const int64_t i = b0 + lane;
        if (i < n) {
            uint4 v;
            if (p.pkts) {
                v = __ldcs(p.pkts + i);
            } else {
                v.x = __ldcs(p.cols.src + i);
                v.y = __ldcs(p.cols.dst + i);
                v.z = ((uint32_t)__ldcs(p.cols.sport + i) << 16) | (uint32_t)__ldcs(p.cols.dport + i);
                v.w = __ldcs(p.cols.proto + i);
            }
            const uint32_t rr[4] = {ms_ip_row(t.ipb[0], t.ipc[0], v.x), ms_ip_row(t.ipb[1], t.ipc[1], v.y),
                                    (uint32_t)__ldg(t.cls + (v.w & 0xFFu)) * t.sp_rows + __ldg(t.port[0] + (v.z >> 16)),
                                    __ldg(t.port[1] + (v.z & 0xFFFFu))};
            PFW_CHECK(rr[0] < t.nrows[0] && rr[1] < t.nrows[1] && rr[2] < t.nrows[2] && rr[3] < t.nrows[3]);
            s_row[warp][lane] = make_uint4(rr[0], rr[1], rr[2], rr[3]);
            uint4 hq[4];  // each dimension's head entry: the first 8 blocks' u16 line indices
#pragma unroll
            for (int d = 0; d < 4; d++)
                hq[d] = __ldg(reinterpret_cast<const uint4 *>(u.head + u.head_off[d] + (size_t)rr[d] * 8));
#pragma unroll
            for (int j = 0; j < K; j++) {
                uint32_t l[4];
#pragma unroll
                for (int d = 0; d < 4; d++) {
                    const uint32_t h2 = (j >> 1) == 0 ? hq[d].x : (j >> 1) == 1 ? hq[d].y : (j >> 1) == 2 ? hq[d].z : hq[d].w;
                    l[d] = ((h2 >> (16 * (j & 1))) & 0xFFFFu) + (CP ? 0u : __ldg(u.loff + d * u.nblk + j));
                }
                if constexpr (CP) s_ln[warp][lane][j] = make_uint2(l[0] | (l[1] << 16), l[2] | (l[3] << 16));
                else s_ln[warp][lane][j] = make_uint4(l[0], l[1], l[2], l[3]);
            }
        }
        s_res[warp][lane] = PFW_NO_MATCH;
        __syncwarp();
        if (nsteps > 0) {
            int pj = grp < nv ? grp : -1;
            int next = P;
            int s = 0, slot = 0;  // block, and its slot in the packet's parked window
            uint4 q = pj >= 0 ? line4(s_ln[warp][pj][0], 0u) : zq;
            while (next < nv + P) {
                uint32_t w[4][V];
                ms_load_rows<V>(lines + ((size_t)q.x << 5) + lv, lines + ((size_t)q.y << 5) + lv,
                                lines + ((size_t)q.z << 5) + lv, lines + ((size_t)q.w << 5) + lv, w);
                uint32_t x[V], any = 0u;
#pragma unroll
                for (int k = 0; k < V; k++) {
                    x[k] = w[0][k] & w[1][k] & w[2][k] & w[3][k];
                    any |= x[k];
                }
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, any != 0u);
                const unsigned gbits = (bal >> gbase) & ((1u << G) - 1u);
                if (any != 0u && (gbits & below) == 0u) {  // park the words; the bit is resolved after the loop
                    s_res[warp][pj] = (uint32_t)s * 32u + lv;
                    uint4 *px = reinterpret_cast<uint4 *>(&s_ln[warp][pj][0]);
#pragma unroll
                    for (int k = 0; k < V; k += 4) px[k / 4] = make_uint4(x[k], x[k + 1], x[k + 2], x[k + 3]);
                }
                const bool act = pj >= 0;
                const bool done = act && (gbits != 0u || s + 1 >= nsteps);
                const unsigned dm = __ballot_sync(0xFFFFFFFFu, done && gl == 0);
                const int np = next + __popc(dm & groups_below);
                const bool take = np < nv;
                // the next block's line numbers: a new packet's block 0, or this
                // packet's next parked block (one shared 16-byte load either way)
                const int ns = done ? 0 : s + (act ? 1 : 0);
                const int nslot = done ? 0 : (act ? (slot + 1 == K ? 0 : slot + 1) : slot);
                // past the parked window (rare): the group parks the next K
                // blocks' line numbers, one block per lane (one round trip per
                // K blocks instead of one per block)
                const bool repark = act && !done && nslot == 0;
                if (__any_sync(0xFFFFFFFFu, repark)) {
                    for (int j = gl; repark && j < K && ns + j < nsteps; j += G) {
                        const uint4 rw = s_row[warp][pj];
                        const uint32_t b = (uint32_t)(ns + j);
                        const uint32_t i0 = __ldg(u.ptr + u.ptr_off[0] + (size_t)rw.x * u.pstride + b);
                        const uint32_t i1 = __ldg(u.ptr + u.ptr_off[1] + (size_t)rw.y * u.pstride + b);
                        const uint32_t i2 = __ldg(u.ptr + u.ptr_off[2] + (size_t)rw.z * u.pstride + b);
                        const uint32_t i3 = __ldg(u.ptr + u.ptr_off[3] + (size_t)rw.w * u.pstride + b);
                        if constexpr (CP)
                            s_ln[warp][pj][j] = make_uint2(i0 | (i1 << 16), i2 | (i3 << 16));
                        else
                            s_ln[warp][pj][j] = make_uint4(__ldg(u.loff + b) + i0, __ldg(u.loff + u.nblk + b) + i1,
                                                           __ldg(u.loff + 2 * u.nblk + b) + i2,
                                                           __ldg(u.loff + 3 * u.nblk + b) + i3);
                    }
                    __syncwarp();
                }
                const int qi = done ? (np & 31) : (pj & 31);
                const uint4 qn = line4(s_ln[warp][qi][nslot], (uint32_t)ns);
                q = (done && !take) || !act ? zq : qn;
                s = ns;
                slot = nslot;
                pj = done ? (take ? np : -1) : pj;
                next += __popc(dm);
            }
        }
        __syncwarp();
        if (i < n) {
            uint32_t res = s_res[warp][lane];
            if (res != PFW_NO_MATCH) res = ms_parked_first_bit<V>(reinterpret_cast<const uint4 *>(&s_ln[warp][lane][0]), res);
            PFW_CHECK(res == PFW_NO_MATCH || (res >= p.lo && res < p.hi));
            emit_result<MODE, true>(p, (uint32_t)i, res, span, st_sum, st_max);
        }
        __syncwarp();
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

// Lean scan of whole-table windows with BLOCK SUMMARIES over compressed rows
// (the adversarial config: most blocks hold no rule that can match a packet
// on every field).  Lookup phase (one packet per lane): the packet's
// candidate blocks -- set bits of the AND of its four summary rows -- and the
// four line numbers of the first MS_SUM_PARK of them, parked in shared memory
// (one 16-byte entry per candidate, the zero line past the last one).  The
// step loop then walks each packet's list like the lean kernels walk steps:
// one candidate block per group per iteration, the first-match bit resolved
// after the loop.  A packet with more candidates than parked ones whose
// parked blocks all fail continues after the loop, one packet per lane, with
// the summary search over the remaining blocks (rare: the parked list covers
// the adversarial recipe's tail).
#ifndef MS_SUM_PARK
#define MS_SUM_PARK 6
#endif
#ifndef MS_SUM_LO_BLOCKS
#define MS_SUM_LO_BLOCKS 64  // (1 KB of shared memory: rulesets up to 64K rules)
#endif
template <int MODE, int MINB>
__global__ void __launch_bounds__(MS_BLOCK, MINB)
    ms_lean_sum_kernel(ScanParams p, MsView t, MsCmp u, uint32_t zline) {
    constexpr int G = 8, V = 4, P = 4, K = MS_SUM_PARK;
    // per packet: the candidates' line numbers (the matching candidate's
    // entry is reused for the finding lane's AND words), blocks, count
    __shared__ uint4 s_cl[MS_BLOCK / 32][32][K];
    __shared__ uint16_t s_cb[MS_BLOCK / 32][32][K];
    __shared__ uint4 s_lo[MS_SUM_LO_BLOCKS];  // loff of block b (x..w = dimension), when nblk <= MS_SUM_LO_BLOCKS
    __shared__ uint8_t s_nc[MS_BLOCK / 32][32];  // candidates parked | (more << 7)
    __shared__ uint32_t s_res[MS_BLOCK / 32][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / G, gl = lane % G, gbase = grp * G;
    const uint32_t lv = (uint32_t)gl * V;
    const unsigned below = (1u << gl) - 1u;
    const unsigned groups_below = (1u << gbase) - 1u;
    const int64_t gw = ((int64_t)blockIdx.x * MS_BLOCK + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * MS_BLOCK) >> 5;
    const int64_t n = p.n;
    const uint32_t span = (uint32_t)(p.win_hi > p.win_lo ? p.win_hi - p.win_lo : 0);
    const bool empty = p.lo >= p.hi;
    const uint32_t kb1 = empty ? 0u : (uint32_t)((p.hi - 1) >> 10);  // last block of the window
    const uint32_t *lines = u.lines;
    const uint4 zq = make_uint4(zline, zline, zline, zline);
    unsigned long long st_sum = 0, st_blocks = 0;
    unsigned st_max = 0;
    const bool lo_sh = u.nblk <= MS_SUM_LO_BLOCKS;  // the parking loop reads loff from shared memory
    if (lo_sh) {
        for (int b = threadIdx.x; b < (int)u.nblk; b += MS_BLOCK)
            s_lo[b] = make_uint4(__ldg(u.loff + b), __ldg(u.loff + u.nblk + b), __ldg(u.loff + 2 * u.nblk + b),
                                 __ldg(u.loff + 3 * u.nblk + b));
        __syncthreads();
    }

    for (int64_t b0 = gw * 32; b0 < n; b0 += nw * 32) {
        const int nv = (int)((n - b0) < 32 ? (n - b0) : 32);
        const int64_t i = b0 + lane;
        int nc = 0, more = 0;
        if (i < n && !empty) {
            uint4 v;
            if (p.pkts) {
                v = __ldcs(p.pkts + i);
            } else {
                v.x = __ldcs(p.cols.src + i);
                v.y = __ldcs(p.cols.dst + i);
                v.z = ((uint32_t)__ldcs(p.cols.sport + i) << 16) | (uint32_t)__ldcs(p.cols.dport + i);
                v.w = __ldcs(p.cols.proto + i);
            }
            const uint32_t rr[4] = {ms_ip_row(t.ipb[0], t.ipc[0], v.x), ms_ip_row(t.ipb[1], t.ipc[1], v.y),
                                    (uint32_t)__ldg(t.cls + (v.w & 0xFFu)) * t.sp_rows + __ldg(t.port[0] + (v.z >> 16)),
                                    __ldg(t.port[1] + (v.z & 0xFFFFu))};
            PFW_CHECK(rr[0] < t.nrows[0] && rr[1] < t.nrows[1] && rr[2] < t.nrows[2] && rr[3] < t.nrows[3]);
            // the candidates' line indices come 8 blocks (16 bytes) per load and
            // dimension: a packet's candidates cluster, so one chunk serves several
            uint4 ch[4];
            uint32_t cc = 0xFFFFFFFFu;  // chunk (block / 8) held in ch
            for (uint32_t w = 0; w <= kb1 / 32u && !more; w++) {
                uint32_t a = __ldg(u.sum[0] + (size_t)rr[0] * u.sw + w) & __ldg(u.sum[1] + (size_t)rr[1] * u.sw + w) &
                             __ldg(u.sum[2] + (size_t)rr[2] * u.sw + w) & __ldg(u.sum[3] + (size_t)rr[3] * u.sw + w);
                const int rel1 = (int)kb1 - 32 * (int)w;
                a &= rel1 >= 31 ? 0xFFFFFFFFu : ((2u << rel1) - 1u);
                while (a) {
                    if (nc == K) {
                        more = 1;
                        break;
                    }
                    const uint32_t b = 32u * w + (uint32_t)(__ffs(a) - 1);
                    a &= a - 1u;
                    if ((b >> 3) != cc) {
                        cc = b >> 3;
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            ch[d] = __ldg(reinterpret_cast<const uint4 *>(
                                b < 8u ? u.head + u.head_off[d] + (size_t)rr[d] * 8
                                       : u.ptr + u.ptr_off[d] + (size_t)rr[d] * u.pstride + 8u * cc));
                    }
                    uint32_t q[4];
                    const uint32_t wi = (b >> 1) & 3u, sh = 16u * (b & 1u);
                    uint4 lo4;
                    if (lo_sh) lo4 = s_lo[b];
                    else lo4 = make_uint4(__ldg(u.loff + b), __ldg(u.loff + u.nblk + b), __ldg(u.loff + 2 * u.nblk + b),
                                          __ldg(u.loff + 3 * u.nblk + b));
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        const uint32_t h2 = wi == 0 ? ch[d].x : wi == 1 ? ch[d].y : wi == 2 ? ch[d].z : ch[d].w;
                        q[d] = (d == 0 ? lo4.x : d == 1 ? lo4.y : d == 2 ? lo4.z : lo4.w) + ((h2 >> sh) & 0xFFFFu);
                    }
                    s_cl[warp][lane][nc] = make_uint4(q[0], q[1], q[2], q[3]);
                    s_cb[warp][lane][nc] = (uint16_t)b;
                    nc++;
                }
            }
        }
        if (nc == 0) s_cl[warp][lane][0] = zq;  // an empty list: its first entry is the zero line
        s_nc[warp][lane] = (uint8_t)(nc | (more << 7));
        s_res[warp][lane] = PFW_NO_MATCH;
        __syncwarp();
        {
            // group state: packet pj (-1 idle), candidate ck of its list, the
            // candidate's four line numbers q (+ this lane's words)
            int pj = grp < nv ? grp : -1;
            int next = P;
            int ck = 0;
            uint4 q = pj >= 0 ? s_cl[warp][pj][0] : zq;
            int pnc = pj >= 0 ? (int)(s_nc[warp][pj] & 0x7F) : 0;
            while (next < nv + P) {
                uint32_t w[4][V];
                ms_load_rows<V>(lines + ((size_t)q.x << 5) + lv, lines + ((size_t)q.y << 5) + lv,
                                lines + ((size_t)q.z << 5) + lv, lines + ((size_t)q.w << 5) + lv, w);
                uint32_t x[V], any = 0u;
#pragma unroll
                for (int k = 0; k < V; k++) {
                    x[k] = w[0][k] & w[1][k] & w[2][k] & w[3][k];
                    any |= x[k];
                }
                const unsigned bal = __ballot_sync(0xFFFFFFFFu, any != 0u);
                const unsigned gbits = (bal >> gbase) & ((1u << G) - 1u);
                const bool act = pj >= 0;
                if (any != 0u && (gbits & below) == 0u) {  // park the words: the bit is resolved after the loop
                    // block, list slot, lane words (< 2^31: never PFW_NO_MATCH)
                    s_res[warp][pj] = ((uint32_t)s_cb[warp][pj][ck] << 8) | (uint32_t)ck | (lv << 24);
                    s_cl[warp][pj][ck] = make_uint4(x[0], x[1], x[2], x[3]);
                }
                if (act && gl == 0 && p.blocks_read) st_blocks++;
                // done: matched, or the parked list is exhausted (the fallback
                // after the loop takes packets with more candidates)
                const bool done = act && (gbits != 0u || ck + 1 >= pnc);
                const unsigned dm = __ballot_sync(0xFFFFFFFFu, done && gl == 0);
                const int np = next + __popc(dm & groups_below);
                const bool take = np < nv;
                // the next candidate: a new packet's first, or this packet's next
                // (an empty list's first entry is the zero line: it ends at once)
                const int ci = done ? (take ? np : 0) : (pj & 31);
                const int cj = done ? 0 : ck + 1;
                const uint4 qn = s_cl[warp][ci][cj < K ? cj : 0];
                const bool idle_next = done ? !take : !act;
                q = idle_next ? zq : qn;
                pnc = done ? (take ? (int)(s_nc[warp][np] & 0x7F) : 0) : pnc;
                ck = cj;
                pj = done ? (take ? np : -1) : pj;
                next += __popc(dm);
            }
        }
        __syncwarp();
        if (i < n) {
            uint32_t res = s_res[warp][lane];
            if (res != PFW_NO_MATCH) {  // (block << 8 | list slot | lv << 24): the parked words' first bit
                const uint32_t blk = (res >> 8) & 0xFFFFu, slot = res & 0xFFu, wl = res >> 24;
                res = ms_parked_first_bit<V>(&s_cl[warp][lane][slot], blk * 32u + wl);
            } else if (s_nc[warp][lane] & 0x80) {
                // more candidates than parked, none of the parked ones matched:
                // continue the summary search after the last parked block, this
                // lane alone, a whole line (32 words) per row and block
                uint4 v;
                if (p.pkts) {
                    v = __ldg(p.pkts + i);
                } else {
                    v.x = __ldg(p.cols.src + i);
                    v.y = __ldg(p.cols.dst + i);
                    v.z = ((uint32_t)__ldg(p.cols.sport + i) << 16) | (uint32_t)__ldg(p.cols.dport + i);
                    v.w = __ldg(p.cols.proto + i);
                }
                const uint32_t rr[4] = {ms_ip_row(t.ipb[0], t.ipc[0], v.x), ms_ip_row(t.ipb[1], t.ipc[1], v.y),
                                        (uint32_t)__ldg(t.cls + (v.w & 0xFFu)) * t.sp_rows + __ldg(t.port[0] + (v.z >> 16)),
                                        __ldg(t.port[1] + (v.z & 0xFFFFu))};
                uint32_t b = (uint32_t)s_cb[warp][lane][K - 1] + 1u;
                for (; b <= kb1 && res == PFW_NO_MATCH; b++) {
                    const uint32_t wsum = b / 32u, bit = 1u << (b % 32u);
                    if (!(__ldg(u.sum[0] + (size_t)rr[0] * u.sw + wsum) & __ldg(u.sum[1] + (size_t)rr[1] * u.sw + wsum) &
                          __ldg(u.sum[2] + (size_t)rr[2] * u.sw + wsum) & __ldg(u.sum[3] + (size_t)rr[3] * u.sw + wsum) & bit))
                        continue;
                    if (p.blocks_read) st_blocks++;
                    const uint32_t *lp[4];
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        const uint16_t ix = b < 8u ? __ldg(u.head + u.head_off[d] + (size_t)rr[d] * 8 + b)
                                                   : __ldg(u.ptr + u.ptr_off[d] + (size_t)rr[d] * u.pstride + b);
                        lp[d] = lines + ((size_t)(__ldg(u.loff + d * u.nblk + b) + ix) << 5);
                    }
                    for (uint32_t wd = 0; wd < 32u; wd++) {
                        const uint32_t xa = __ldg(lp[0] + wd) & __ldg(lp[1] + wd) & __ldg(lp[2] + wd) & __ldg(lp[3] + wd);
                        if (xa) {
                            res = (b * 32u + wd) * 32u + (uint32_t)(__ffs(xa) - 1);
                            break;
                        }
                    }
                }
            }
            PFW_CHECK(res == PFW_NO_MATCH || (res >= p.lo && res < p.hi));
            emit_result<MODE, true>(p, (uint32_t)i, res, span, st_sum, st_max);
        }
        __syncwarp();
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
    if (p.blocks_read) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) st_blocks += __shfl_xor_sync(0xFFFFFFFFu, st_blocks, o);
        if (lane == 0 && st_blocks) atomicAdd(p.blocks_read, st_blocks);
    }
}

void ms_free(MatchSet *m) {
    if (!m) return;
    if (m->d_bits_all) cudaFree(m->d_bits_all);
    if (m->d_lines) cudaFree(m->d_lines);
    if (m->d_loff) cudaFree(m->d_loff);
    if (m->d_ptr_all) cudaFree(m->d_ptr_all);
    if (m->d_head_all) cudaFree(m->d_head_all);
    for (auto *b : m->d_sum)
        if (b) cudaFree(b);
    for (auto *b : m->d_ipb)
        if (b) cudaFree(b);
    for (auto *c : m->d_ipc)
        if (c) cudaFree(c);
    for (auto *q : m->d_port)
        if (q) cudaFree(q);
    for (auto *q : m->d_pbk)
        if (q) cudaFree(q);
    if (m->d_cls) cudaFree(m->d_cls);
    delete m;
}

// Elementary-interval boundaries of an IP field: 0 and, per rule that can
// match at all, base and the first address past its block.
std::vector<uint32_t> ms_ip_bounds(int64_t n, const uint32_t *base, const uint32_t *mask) {
    std::vector<uint32_t> b;
    b.reserve((size_t)(2 * n + 1));
    b.push_back(0u);
    for (int64_t r = 0; r < n; r++) {
        if (base[r] & ~mask[r]) continue;  // never matches: constant on every interval
        b.push_back(base[r]);
        const uint64_t e = (uint64_t)(base[r] | ~mask[r]) + 1;
        if (e < (1ull << 32)) b.push_back((uint32_t)e);
    }
    std::sort(b.begin(), b.end());
    b.erase(std::unique(b.begin(), b.end()), b.end());
    return b;
}

std::vector<uint32_t> ms_port_bounds(int64_t n, const uint16_t *lo, const uint16_t *hi) {
    std::vector<uint32_t> b;
    b.reserve((size_t)(2 * n + 1));
    b.push_back(0u);
    for (int64_t r = 0; r < n; r++) {
        if (lo[r] > hi[r]) continue;
        b.push_back(lo[r]);
        if ((uint32_t)hi[r] + 1 < 65536u) b.push_back((uint32_t)hi[r] + 1);
    }
    std::sort(b.begin(), b.end());
    b.erase(std::unique(b.begin(), b.end()), b.end());
    return b;
}

template <typename T>
cudaError_t ms_upload(T **d, const T *h, size_t count) {
    cudaError_t e = cudaMalloc(d, count * sizeof(T) + 16);
    if (e == cudaSuccess && count) e = cudaMemcpy(*d, h, count * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

// Block summaries (one bit per 1024-rule block per row) and the auto decision:
// the expected fraction of blocks a packet's AND-summary keeps, for packet
// fields uniform over their domains -- per dimension the interval-length-
// weighted fraction of set summary bits, multiplied over the dimensions.
// Random rulesets keep ~100% (every 1024-rule block has some rule matching
// any value), so they scan without; rulesets whose rules cluster (e.g. the
// adversarial recipe's decoys, all in 128.0.0.0/1) skip most blocks.
int ms_summaries(pfw_ruleset *h, const std::vector<uint32_t> &bs, const std::vector<uint32_t> &bd,
                 const std::vector<uint32_t> &bsp, const std::vector<uint32_t> &bdp) {
    MatchSet *m = h->ms;
    const int64_t blocks = m->wp / 32;             // blocks per row (incl. the padding of the last step)
    const int64_t real = (h->n + 1023) / 1024;     // blocks holding rules
    if (!g_ms_summary || real < 2 || blocks > 32 * 8) return PFW_OK;  // 8 lanes x 32 blocks
    const int64_t sw = (blocks + 31) / 32;
    cudaError_t e = cudaSuccess;
    for (int d = 0; d < 4 && e == cudaSuccess; d++) e = cudaMalloc(&m->d_sum[d], ((size_t)m->rows[d] * sw + 8) * 4);
    for (int d = 0; d < 4 && e == cudaSuccess; d++) {
        if (m->cmp)
            ms_sum_cmp_kernel<<<(unsigned)(h->sms * 8), MS_BLOCK>>>(m->d_lines, m->d_loff + d * m->nblk,
                                                                    m->d_ptr_all + m->ptr_off[d], m->pstride,
                                                                    m->rows[d], blocks, sw, m->d_sum[d]);
        else
            ms_sum_kernel<<<(unsigned)(h->sms * 8), MS_BLOCK>>>(m->d_bits[d], m->rows[d], m->wp, sw, m->d_sum[d]);
        g_launches++;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    double keep = 1.0;
    const std::vector<uint32_t> *bnd[4] = {&bs, &bd, &bsp, &bdp};
    for (int d = 0; d < 4 && e == cudaSuccess; d++) {
        std::vector<uint32_t> hs((size_t)m->rows[d] * sw);
        e = cudaMemcpy(hs.data(), m->d_sum[d], hs.size() * 4, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) break;
        const std::vector<uint32_t> &b = *bnd[d];
        const double dom = d < 2 ? 4294967296.0 : 65536.0;
        double acc = 0.0, wsum = 0.0;
        for (int64_t row = 0; row < m->rows[d]; row++) {
            const int64_t i = d == MSD_SPORT ? row % m->sp_rows : row;  // every protocol class weighs alike
            const double len = (i + 1 < (int64_t)b.size() ? (double)b[(size_t)i + 1] : dom) - (double)b[(size_t)i];
            int ones = 0;
            for (int64_t j = 0; j < sw; j++) ones += __builtin_popcount(hs[(size_t)(row * sw + j)]);
            acc += len * ones / (double)real;
            wsum += len;
        }
        keep *= wsum > 0 ? acc / wsum : 1.0;
    }
    if (e != cudaSuccess) {
        for (auto *&q : m->d_sum)
            if (q) cudaFree(q), q = nullptr;
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            return PFW_OK;
        }
        return set_err(PFW_ERR_CUDA, "match-set summaries failed: %s", cudaGetErrorString(e));
    }
    m->sw = sw;
    m->sum_keep = keep;
    m->use_sum = g_ms_summary == 1 || keep < MS_SUM_KEEP_MAX;
    for (int d = 0; d < 4; d++) m->bytes += ((size_t)m->rows[d] * sw + 8) * 4;
    return PFW_OK;
}

// Compressed rows (see MatchSet::cmp): per (dimension, block) the block's own
// boundaries -> its distinct lines (built by the reference predicate on the
// block's rules), and per row and block the index of the row's line.  The
// device rule columns / interval values come from ms_create's build.
// Returns cudaSuccess with m->cmp unset when a block has more than 65536
// lines (u16 indices).
cudaError_t ms_compress_build(pfw_ruleset *h, MatchSet *m, int64_t n, const uint8_t *proto,
                              const uint32_t *src_base, const uint32_t *src_mask, const uint16_t *sport_lo,
                              const uint16_t *sport_hi, const uint32_t *dst_base, const uint32_t *dst_mask,
                              const uint16_t *dport_lo, const uint16_t *dport_hi, int ncls,
                              const uint32_t *d_sb, const uint32_t *d_sm, const uint32_t *d_db,
                              const uint32_t *d_dm, const uint16_t *d_slo, const uint16_t *d_shi,
                              const uint16_t *d_dlo, const uint16_t *d_dhi, const uint8_t *d_pr,
                              const int *d_clsp, uint32_t *const *d_vals, size_t budget) {
    const int64_t nblk = m->wp / 32;
    std::vector<uint32_t> bnd, boff((size_t)(4 * nblk + 1)), loff((size_t)(4 * nblk + 1));
    std::vector<MsLineDesc> desc;
    std::vector<uint32_t> v;
    for (int d = 0; d < 4; d++) {
        for (int64_t b = 0; b < nblk; b++) {
            v.assign(1, 0u);
            const int64_t r0 = b * 1024, r1 = std::min<int64_t>(n, r0 + 1024);
            for (int64_t r = r0; r < r1; r++) {
                if (d < 2) {
                    const uint32_t base = d == MSD_SRC ? src_base[r] : dst_base[r];
                    const uint32_t mask = d == MSD_SRC ? src_mask[r] : dst_mask[r];
                    if (base & ~mask) continue;
                    v.push_back(base);
                    const uint64_t e = (uint64_t)(base | ~mask) + 1;
                    if (e < (1ull << 32)) v.push_back((uint32_t)e);
                } else {
                    const uint32_t lo = d == MSD_SPORT ? sport_lo[r] : dport_lo[r];
                    const uint32_t hi = d == MSD_SPORT ? sport_hi[r] : dport_hi[r];
                    if (lo > hi) continue;
                    v.push_back(lo);
                    if (hi + 1 < 65536u) v.push_back(hi + 1);
                }
            }
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
            const int ncl = d == MSD_SPORT ? ncls : 1;
            if ((int64_t)v.size() * ncl > 65536) return cudaSuccess;  // u16 line indices
            boff[(size_t)(d * nblk + b)] = (uint32_t)bnd.size();
            loff[(size_t)(d * nblk + b)] = (uint32_t)desc.size();
            bnd.insert(bnd.end(), v.begin(), v.end());
            for (int c = 0; c < ncl; c++)
                for (uint32_t x : v) desc.push_back(MsLineDesc{x, (uint32_t)b, (uint16_t)d, (uint16_t)c});
        }
    }
    boff[(size_t)(4 * nblk)] = (uint32_t)bnd.size();
    loff[(size_t)(4 * nblk)] = (uint32_t)desc.size();
    const int64_t pstride = ((nblk + 16 + 7) / 8) * 8;
    size_t need = desc.size() * 128;
    for (int d = 0; d < 4; d++) need += (size_t)m->rows[d] * ((size_t)pstride + 8) * 2;
    if (need > budget) return cudaSuccess;  // over budget even compressed
    m->nblk = nblk;
    m->pstride = pstride;
    m->nlines = (int64_t)desc.size();
    uint32_t *d_bnd = nullptr, *d_boff = nullptr;
    MsLineDesc *d_desc = nullptr;
    cudaError_t e = ms_upload(&d_bnd, bnd.data(), bnd.size());
    if (e == cudaSuccess) e = ms_upload(&d_boff, boff.data(), boff.size());
    loff.resize(loff.size() + 8, loff.back());  // slack: the lookup phase reads 8 entries from any block
    if (e == cudaSuccess) e = ms_upload(&m->d_loff, loff.data(), loff.size());
    if (e == cudaSuccess) e = ms_upload(&d_desc, desc.data(), desc.size());
    if (e == cudaSuccess) e = cudaMalloc(&m->d_lines, ((size_t)m->nlines * 32 + 4 * 32) * 4);
    if (e == cudaSuccess) e = cudaMemset(m->d_lines + (size_t)m->nlines * 32, 0, 4 * 32 * 4);
    size_t pent = 0;
    for (int d = 0; d < 4; d++) {
        m->ptr_off[d] = pent;
        pent += (size_t)m->rows[d] * (size_t)m->pstride;
    }
    if (e == cudaSuccess) e = cudaMalloc(&m->d_ptr_all, (pent + 16) * 2);
    if (e == cudaSuccess) e = cudaMemset(m->d_ptr_all, 0, (pent + 16) * 2);
    size_t hent = 0;
    for (int d = 0; d < 4; d++) {
        m->head_off[d] = hent;
        hent += (size_t)m->rows[d] * 8;
    }
    if (e == cudaSuccess) e = cudaMalloc(&m->d_head_all, (hent + 8) * 2);
    if (e == cudaSuccess) {
        ms_line_kernel<<<(unsigned)(h->sms * 8), MS_BLOCK>>>(d_desc, m->nlines, n, d_sb, d_sm, d_db, d_dm, d_slo,
                                                             d_shi, d_dlo, d_dhi, d_pr, d_clsp, m->d_lines);
        g_launches++;
        for (int d = 0; d < 4; d++) {
            ms_ptr_kernel<<<(unsigned)(h->sms * 8), 256>>>(d_vals[d], m->rows[d], m->sp_rows, d == MSD_SPORT, nblk,
                                                           d_bnd, d_boff + d * nblk, m->d_ptr_all + m->ptr_off[d],
                                                           m->pstride);
            g_launches++;
        }
        // the head array: each row's first 8 indices, dense (one strided copy per dimension)
        for (int d = 0; d < 4 && e == cudaSuccess; d++)
            e = cudaMemcpy2D(m->d_head_all + m->head_off[d], 16, m->d_ptr_all + m->ptr_off[d],
                             (size_t)m->pstride * 2, 16, (size_t)m->rows[d], cudaMemcpyDeviceToDevice);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    for (void *q : {(void *)d_bnd, (void *)d_boff, (void *)d_desc})
        if (q) cudaFree(q);
    if (e == cudaSuccess) m->cmp = true;
    return e;
}

// Build the match sets of ruleset h (host columns as given to
// pfw_ruleset_create).  Tables that would exceed the memory budget are not
// built: the ruleset then scans rule by rule.
int ms_create(pfw_ruleset *h, const uint8_t *proto, const uint32_t *src_base, const uint32_t *src_mask,
              const uint16_t *sport_lo, const uint16_t *sport_hi, const uint32_t *dst_base,
              const uint32_t *dst_mask, const uint16_t *dport_lo, const uint16_t *dport_hi) {
    const int64_t n = h->n;
    if (n == 0 || !g_matchset) return PFW_OK;
    const std::vector<uint32_t> bs = ms_ip_bounds(n, src_base, src_mask);
    const std::vector<uint32_t> bd = ms_ip_bounds(n, dst_base, dst_mask);
    const std::vector<uint32_t> bsp = ms_port_bounds(n, sport_lo, sport_hi);
    const std::vector<uint32_t> bdp = ms_port_bounds(n, dport_lo, dport_hi);
    // protocol classes: one per protocol a rule names, plus one for the rest
    // (their packets match only ANY rules)
    std::vector<int> cls_proto;
    uint8_t cls[256];
    {
        bool named[256] = {};
        for (int64_t r = 0; r < n; r++) named[proto[r]] = true;
        for (int v = 1; v < 256; v++)
            if (named[v]) cls_proto.push_back(v);
        const int other = (int)cls_proto.size();
        for (int v = 0; v < 256; v++) cls[v] = (uint8_t)other;
        for (int c = 0; c < other; c++) cls[cls_proto[(size_t)c]] = (uint8_t)c;
        cls_proto.push_back(-1);
    }
    MatchSet *m = new MatchSet();
    m->wp = (((n + 31) / 32 + 127) / 128) * 128;  // whole 4-word-per-lane steps
    m->sp_rows = (int64_t)bsp.size();
    m->rows[MSD_SRC] = (int64_t)bs.size();
    m->rows[MSD_DST] = (int64_t)bd.size();
    m->rows[MSD_SPORT] = (int64_t)cls_proto.size() * m->sp_rows;
    m->rows[MSD_DPORT] = (int64_t)bdp.size();
    size_t bytes = 0;
    for (int d = 0; d < 4; d++) bytes += (size_t)m->rows[d] * (size_t)m->wp * 4;
    bytes += (bs.size() + bd.size()) * 4 + 2 * 65537 * 4 + 2 * 65536 * 2 + 256;
    m->bytes = bytes;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
    const size_t budget = g_ms_budget_mb > 0 ? (size_t)g_ms_budget_mb << 20 : free_b / 4;
    bool fits = bytes <= budget;
    uint64_t all_words = 0;  // word offsets from the common base are 32-bit in the scan
    for (int d = 0; d < 4; d++) all_words += (uint64_t)m->rows[d] * (uint64_t)m->wp + 4 * 32;
    fits = fits && all_words < (1ull << 32);
    // compressed rows: forced, or (auto) for large rulesets or when the plain
    // rows do not fit -- ~20x smaller; slower than plain rows only while
    // those stay L2-friendly (<= 16K rules)
    const bool use_cmp = g_ms_compress == 1 || (g_ms_compress == 2 && (!fits || n > MS_CMP_MIN_RULES));
    // (boundary indices are packed in 24 bits: beyond ~8M rules the ruleset scans rule by rule)
    if ((!fits && !use_cmp) || bs.size() >= (1u << 24) || bd.size() >= (1u << 24)) {
        delete m;
        return PFW_OK;  // too large for the budget: rule-by-rule scan
    }
    // lookup tables
    std::vector<uint4> ipc[2];
    const std::vector<uint32_t> *ipb[2] = {&bs, &bd};
    for (int d = 0; d < 2; d++) {
        const std::vector<uint32_t> &b = *ipb[d];
        std::vector<uint32_t> c(65537);
        size_t k = 0;
        for (uint32_t blk = 0; blk < 65536; blk++) {
            while (k < b.size() && b[k] < (blk << 16)) k++;
            c[blk] = (uint32_t)k;
        }
        c[65536] = (uint32_t)b.size();
        ipc[d].resize(65537);
        for (uint32_t blk = 0; blk <= 65536; blk++) {
            const uint32_t cnt = blk < 65536 ? c[blk + 1] - c[blk] : 0u;
            uint16_t h[6];
            for (uint32_t k = 0; k < 6; k++) h[k] = k < cnt ? (uint16_t)(b[c[blk] + k] & 0xFFFFu) : (uint16_t)0xFFFFu;
            ipc[d][blk] = make_uint4(c[blk] | ((cnt < 255u ? cnt : 255u) << 24), h[0] | ((uint32_t)h[1] << 16),
                                     h[2] | ((uint32_t)h[3] << 16), h[4] | ((uint32_t)h[5] << 16));
        }
    }
    std::vector<uint16_t> ptab[2];
    const std::vector<uint32_t> *pb[2] = {&bsp, &bdp};
    for (int d = 0; d < 2; d++) {
        ptab[d].resize(65536);
        size_t k = 0;
        for (uint32_t v = 0; v < 65536; v++) {
            while (k + 1 < pb[d]->size() && (*pb[d])[k + 1] <= v) k++;
            ptab[d][v] = (uint16_t)k;  // (port intervals <= 65536)
        }
    }
    // device copies of the rule columns (build only)
    uint32_t *d_sb = nullptr, *d_sm = nullptr, *d_db = nullptr, *d_dm = nullptr, *d_vals[4] = {};
    uint16_t *d_slo = nullptr, *d_shi = nullptr, *d_dlo = nullptr, *d_dhi = nullptr;
    uint8_t *d_pr = nullptr;
    int *d_clsp = nullptr;
    cudaError_t e = cudaSuccess;
    // one allocation for the four dimensions (the scan addresses every row
    // from one base); + one 4-word-per-lane step of padding after each: the
    // last step of a row may read past its end (masked), also on a last row
    if (!use_cmp) {
        size_t words = 0;
        for (int d = 0; d < 4; d++) words += (size_t)m->rows[d] * (size_t)m->wp + 4 * 32;
        e = cudaMalloc(&m->d_bits_all, words * 4);
        size_t off = 0;
        for (int d = 0; d < 4 && e == cudaSuccess; d++) {
            m->d_bits[d] = m->d_bits_all + off;
            off += (size_t)m->rows[d] * (size_t)m->wp;
            e = cudaMemsetAsync(m->d_bits_all + off, 0, 4 * 32 * 4);
            off += 4 * 32;
        }
    }
    if (e == cudaSuccess) e = ms_upload(&m->d_ipb[0], bs.data(), bs.size());
    if (e == cudaSuccess) e = ms_upload(&m->d_ipb[1], bd.data(), bd.size());
    if (e == cudaSuccess) e = ms_upload(&m->d_ipc[0], ipc[0].data(), ipc[0].size());
    if (e == cudaSuccess) e = ms_upload(&m->d_ipc[1], ipc[1].data(), ipc[1].size());
    if (e == cudaSuccess) e = ms_upload(&m->d_port[0], ptab[0].data(), ptab[0].size());
    if (e == cudaSuccess) e = ms_upload(&m->d_port[1], ptab[1].data(), ptab[1].size());
    // port buckets of 32 ports: interval(p) = base[p >> 5] + popc(bits[p >> 5]
    // & ones up to bit p & 31) -- 12 KB per dimension (2048 u32 boundary-bit
    // words, then 2048 u16 bases), small enough to stay in L1
    for (int d = 0; d < 2 && e == cudaSuccess; d++) {
        std::vector<uint32_t> bk(3072, 0u);
        for (uint32_t b = 0; b < 2048; b++) {
            uint32_t bits = 0;
            for (uint32_t j = 1; j < 32; j++)
                if (ptab[d][b * 32 + j] != ptab[d][b * 32 + j - 1]) bits |= 1u << j;
            bk[b] = bits;
            bk[2048 + b / 2] |= (uint32_t)ptab[d][b * 32] << (16 * (b & 1));
        }
        e = ms_upload(&m->d_pbk[d], bk.data(), bk.size());
    }
    if (e == cudaSuccess) e = ms_upload(&m->d_cls, cls, 256);
    if (e == cudaSuccess) e = ms_upload(&d_sb, src_base, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_sm, src_mask, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_db, dst_base, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_dm, dst_mask, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_slo, sport_lo, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_shi, sport_hi, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_dlo, dport_lo, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_dhi, dport_hi, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_pr, proto, (size_t)n);
    if (e == cudaSuccess) e = ms_upload(&d_clsp, cls_proto.data(), cls_proto.size());
    if (e == cudaSuccess) e = ms_upload(&d_vals[0], bs.data(), bs.size());
    if (e == cudaSuccess) e = ms_upload(&d_vals[1], bd.data(), bd.size());
    if (e == cudaSuccess) e = ms_upload(&d_vals[2], bsp.data(), bsp.size());
    if (e == cudaSuccess) e = ms_upload(&d_vals[3], bdp.data(), bdp.size());
    if (e == cudaSuccess && !use_cmp) {
        MsBuildArgs a{};
        a.n = n;
        a.wp = m->wp;
        a.proto = d_pr;
        a.cls_proto = d_clsp;
        a.ivl = m->sp_rows;
        const unsigned grid = (unsigned)(h->sms * 8);
        for (int d = 0; d < 4; d++) {
            a.rows = m->rows[d];
            a.vals = d_vals[d];
            a.bits = m->d_bits[d];
            a.base = d == MSD_SRC ? d_sb : d_db;
            a.mask = d == MSD_SRC ? d_sm : d_dm;
            a.lo = d == MSD_SPORT ? d_slo : d_dlo;
            a.hi = d == MSD_SPORT ? d_shi : d_dhi;
            switch (d) {
                case MSD_SRC: ms_build_kernel<MSD_SRC><<<grid, MS_BLOCK>>>(a); break;
                case MSD_DST: ms_build_kernel<MSD_DST><<<grid, MS_BLOCK>>>(a); break;
                case MSD_SPORT: ms_build_kernel<MSD_SPORT><<<grid, MS_BLOCK>>>(a); break;
                default: ms_build_kernel<MSD_DPORT><<<grid, MS_BLOCK>>>(a); break;
            }
            g_launches++;
        }
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (e == cudaSuccess && use_cmp) {
        e = ms_compress_build(h, m, n, proto, src_base, src_mask, sport_lo, sport_hi, dst_base, dst_mask, dport_lo,
                              dport_hi, (int)cls_proto.size(), d_sb, d_sm, d_db, d_dm, d_slo, d_shi, d_dlo, d_dhi,
                              d_pr, d_clsp, d_vals, budget);
        if (e == cudaSuccess && !m->cmp) e = cudaErrorMemoryAllocation;  // not compressible / over budget
    }
    // summaries (from whichever rows were built); when the scan will use them
    // (rules clustered enough to skip blocks), auto also compresses plain rows:
    // the summary scan visits few, scattered blocks, which the compressed
    // rows' small footprint keeps in L2 (adversarial config: +9%)
    int src = PFW_OK;
    if (e == cudaSuccess) {
        h->ms = m;
        src = ms_summaries(h, bs, bd, bsp, bdp);
        h->ms = nullptr;
        if (src == PFW_OK && !m->cmp && m->use_sum && g_ms_compress == 2) {
            const cudaError_t ec = ms_compress_build(h, m, n, proto, src_base, src_mask, sport_lo, sport_hi, dst_base,
                                                     dst_mask, dport_lo, dport_hi, (int)cls_proto.size(), d_sb, d_sm,
                                                     d_db, d_dm, d_slo, d_shi, d_dlo, d_dhi, d_pr, d_clsp, d_vals,
                                                     budget);
            if (ec == cudaSuccess && m->cmp) {  // drop the plain rows
                cudaFree(m->d_bits_all);
                m->d_bits_all = nullptr;
                for (auto *&q : m->d_bits) q = nullptr;
            } else {  // optional: keep the plain rows
                cudaGetLastError();
                for (void *q : {(void *)m->d_lines, (void *)m->d_loff, (void *)m->d_ptr_all, (void *)m->d_head_all})
                    if (q) cudaFree(q);
                m->d_lines = nullptr;
                m->d_loff = nullptr;
                m->d_ptr_all = nullptr;
                m->d_head_all = nullptr;
                m->cmp = false;
            }
        }
    }
    for (void *q : {(void *)d_sb, (void *)d_sm, (void *)d_db, (void *)d_dm, (void *)d_slo, (void *)d_shi,
                    (void *)d_dlo, (void *)d_dhi, (void *)d_pr, (void *)d_clsp, (void *)d_vals[0],
                    (void *)d_vals[1], (void *)d_vals[2], (void *)d_vals[3]})
        if (q) cudaFree(q);
    if (e != cudaSuccess) {
        ms_free(m);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            return PFW_OK;  // could not place the tables: rule-by-rule scan
        }
        return set_err(PFW_ERR_CUDA, "match-set build failed: %s", cudaGetErrorString(e));
    }
    if (src != PFW_OK) {
        ms_free(m);
        return src;
    }
    if (m->cmp) {  // account the compressed rows instead of the plain ones
        size_t plain = 0;
        for (int d = 0; d < 4; d++) plain += (size_t)m->rows[d] * (size_t)m->wp * 4;
        m->bytes -= plain;
        m->bytes += ((size_t)m->nlines * 32 + 4 * 32) * 4 + (size_t)(4 * m->nblk + 1) * 4;
        for (int d = 0; d < 4; d++) m->bytes += (size_t)m->rows[d] * ((size_t)m->pstride + 8) * 2;
    }
    h->ms = m;
    return PFW_OK;
}

static MsView ms_view(const MatchSet *m) {
    MsView t{};
    t.bits0 = m->d_bits_all;
    for (int d = 0; d < 4; d++) t.off[d] = (uint32_t)(m->d_bits[d] - m->d_bits_all);
#ifdef PFW_CHECKS
    for (int d = 0; d < 4; d++) t.nrows[d] = (uint32_t)m->rows[d];
    t.words = 0;
    for (int d = 0; d < 4; d++) t.words += (uint64_t)m->rows[d] * (uint64_t)m->wp + 4 * 32;
#endif
    t.ipb[0] = m->d_ipb[0];
    t.ipb[1] = m->d_ipb[1];
    t.ipc[0] = m->d_ipc[0];
    t.ipc[1] = m->d_ipc[1];
    t.port[0] = m->d_port[0];
    t.port[1] = m->d_port[1];
    t.pbk[0] = m->d_pbk[0];
    t.pbk[1] = m->d_pbk[1];
    t.cls = m->d_cls;
    t.wp = m->wp;
    t.sp_rows = (uint32_t)m->sp_rows;
    return t;
}

template <int MODE>
int launch_ms_k(pfw_ruleset *h, const ScanParams &p, cudaStream_t st) {
    const MatchSet *m = h->ms;
    const MsView t = ms_view(m);
    MsSum u{};
    for (int d = 0; d < 4; d++) u.sum[d] = m->d_sum[d];
    u.sw = (uint32_t)m->sw;
    MsCmp uc{};
    for (int d = 0; d < 4; d++) uc.sum[d] = m->d_sum[d];
    uc.sw = (uint32_t)m->sw;
    uc.pstride = (uint32_t)m->pstride;
    uc.nblk = (uint32_t)m->nblk;
    uc.ptr = m->d_ptr_all;
    for (int d = 0; d < 4; d++) uc.ptr_off[d] = m->ptr_off[d];
    uc.lines = m->d_lines;
    uc.loff = m->d_loff;
    uc.head = m->d_head_all;
    for (int d = 0; d < 4; d++) uc.head_off[d] = m->head_off[d];
    void (*kern)(ScanParams, MsView, MsNoSum) = nullptr;
    void (*kern_s)(ScanParams, MsView, MsSum) = nullptr;
    void (*kern_c)(ScanParams, MsView, MsCmp) = nullptr;
    // (rows not a whole number of steps long: mask the last step's words)
    const bool win = !(p.lo == 0 && p.hi == h->n) ||
                     (m->wp % ((int64_t)(g_ms_group ? g_ms_group : (h->n > 16384 && !m->cmp ? 16 : 8)) * g_ms_words)) != 0;
    // auto: 8 lanes (4 packets in flight, 1024-rule steps) while the rows'
    // leading lines fit in L2; 16 lanes (2048-rule steps, fewer iterations)
    // for large plain rulesets whose scans run long and mostly miss L2
    const int grp = g_ms_group ? g_ms_group : (h->n > 16384 && !m->cmp ? 16 : 8);
    // block summaries / compressed rows: one step = one 1024-rule block (8 lanes x 4 words)
    const bool sum = m->use_sum && m->sw > 0 && g_ms_summary != 0 &&
                     (m->cmp || (g_ms_words == 4 && (g_ms_group == 0 || g_ms_group == 8)));
    // (compressed rows always scan on 8 lanes x 4 words: one step = one block)
#define PFW_MS_PICK(G_, V_)                                                                     \
    if (grp == G_ && g_ms_words == V_)                                                   \
        kern = win ? ms_scan_kernel<MODE, G_, V_, true> : ms_scan_kernel<MODE, G_, V_, false>;
    PFW_MS_PICK(8, 4)
    PFW_MS_PICK(8, 2)
    PFW_MS_PICK(16, 4)
    PFW_MS_PICK(16, 2)
    PFW_MS_PICK(32, 2)
    PFW_MS_PICK(32, 1)
#undef PFW_MS_PICK
    if (m->cmp) {
        kern = nullptr;
        if (sum) kern_c = win ? ms_scan_kernel<MODE, 8, 4, true, true, true> : ms_scan_kernel<MODE, 8, 4, false, true, true>;
        else kern_c = win ? ms_scan_kernel<MODE, 8, 4, true, false, true> : ms_scan_kernel<MODE, 8, 4, false, false, true>;
    } else if (sum) {
        kern = nullptr;
        kern_s = win ? ms_scan_kernel<MODE, 8, 4, true, true> : ms_scan_kernel<MODE, 8, 4, false, true>;
    }
    if (!kern && !kern_s && !kern_c)
        return set_err(PFW_ERR_INVALID, "ms_group %d x ms_words %d not built", grp, g_ms_words);
    // whole-table scans over plain rows in the default shape: the lean kernel
    void (*kern_l)(ScanParams, MsView, uint32_t) = nullptr;
    // (auto, measured on B200: 4-lane groups with 256-bit loads -- twice the
    // packets in flight per warp -- for batches that fill the GPU only a few
    // times over: under 768K packets (10K rules x 100K packets 3.7 vs 2.1 Gpps,
    // x 512K 7.6 vs 7.3), under 4Mi for rulesets up to 2K rules (the oracle
    // config 6.4 vs 5.5); otherwise 8-lane groups with 64-packet batches: data
    // 13.65 Gpps vs 12.55 on the general kernel, grid 16.15, 1K rules x 16Mi
    // packets 27.9 vs 25.7, 10K rules x 1Mi packets 10.3 vs 9.4)
    const bool small_batch = p.n < (int64_t(3) << 18) || (h->n <= 2048 && p.n < (int64_t(1) << 22));
    const int lean = g_ms_lean == 3 ? (small_batch ? 2 : 6) : g_ms_lean;
    // compressed rows, whole table, no summaries: the lean compressed kernel
    // (tuning ms_lean_cmp: 0 off, 1 8-lane groups, 2 4-lane groups / 256-bit loads)
    void (*kern_lc)(ScanParams, MsView, MsCmp, uint32_t) = nullptr;
    // (default 3: 8-lane groups with u16 parked indices; batches under 192K
    // packets -- a fraction of one wave -- take the 4-lane groups: 100K packets
    // x 100K rules 3.05 vs 2.74 Gpps, equal at 256K, 8.4 vs 6.9 at 1Mi)
    if (g_ms_lean_cmp && kern_c && !sum && !win)
        kern_lc = (g_ms_lean_cmp == 2 || (g_ms_lean_cmp == 3 && p.n < (int64_t(3) << 16))) ? ms_lean_cmp_kernel<MODE, 4>
                  : (g_ms_lean_cmp == 3 && m->nblk <= MS_CP_BLOCKS) ? ms_lean_cmp_kernel<MODE, 8, true>
                                                                     : ms_lean_cmp_kernel<MODE, 8>;
    // block summaries over compressed rows, whole table: the lean candidate walk
    if (g_ms_lean_sum && kern_c && sum && !win)
        kern_lc = g_ms_lean_sum == 2 ? ms_lean_sum_kernel<MODE, 4> : ms_lean_sum_kernel<MODE, PFW_MS_MINB>;
    if (lean && kern && !win && grp == 8 && g_ms_words == 4)
        switch (lean) {
            // 1: 8-lane groups, 1024-rule steps, 32-packet batches
            case 1: kern_l = ms_lean_kernel<MODE, 8, 4, 1, PFW_MS_MINB>; break;
            // 2: 4-lane groups, 256-bit loads, 1024-rule steps, 8 packets per warp
            case 2: kern_l = ms_lean_kernel<MODE, 4, 8, 1, 4>; break;
            // 4: 4-lane groups, 512-rule steps (half the bytes per step), 8 packets per warp
            case 4: kern_l = ms_lean_kernel<MODE, 4, 4, 1, PFW_MS_MINB>; break;
            // 5: as 1 at 6 resident blocks per SM (42 registers)
            case 5: kern_l = ms_lean_kernel<MODE, 8, 4, 1, 6>; break;
            // 6: as 1 with 64-packet batches (half the batch boundaries)
            case 6: kern_l = ms_lean_kernel<MODE, 8, 4, 2, PFW_MS_MINB>; break;
            default: break;
        }
    int occ = g_ctas_per_sm;
    if (occ <= 0) {
        if (kern_l) CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern_l, MS_BLOCK, 0));
        else if (kern_c) CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern_c, MS_BLOCK, 0));
        else if (kern_s) CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern_s, MS_BLOCK, 0));
        else CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, MS_BLOCK, 0));
        if (occ < 1) occ = 1;
    }
    int64_t grid = (int64_t)h->sms * occ;
    const int64_t need = (p.n + MS_BLOCK * PFW_MS_LPB - 1) / (MS_BLOCK * PFW_MS_LPB);  // one batch per warp
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    ScanParams pc = p;
    if ((kern_s || (kern_c && sum)) && g_count_blocks) {
        if (!g_counter_dev) {
            CUDA_TRY(cudaMalloc(&g_counter_dev, sizeof(unsigned long long)));
            CUDA_TRY(cudaMemset(g_counter_dev, 0, sizeof(unsigned long long)));
        }
        pc.blocks_read = g_counter_dev;
    }
    if (kern_lc) {
        if (g_ctas_per_sm <= 0) {
            int o2 = 1;
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, kern_lc, MS_BLOCK, 0));
            grid = std::min<int64_t>((int64_t)h->sms * std::max(o2, 1), need);
        }
        kern_lc<<<(unsigned)grid, MS_BLOCK, 0, st>>>(sum ? pc : p, t, uc, (uint32_t)m->nlines);
    } else if (kern_l) {
        // word offset of the zero padding after the src rows (idle groups read it)
        const uint32_t zoff = (uint32_t)((m->d_bits[0] - m->d_bits_all) + m->rows[0] * m->wp);
        kern_l<<<(unsigned)grid, MS_BLOCK, 0, st>>>(p, t, zoff);
    } else if (kern_c) kern_c<<<(unsigned)grid, MS_BLOCK, 0, st>>>(pc, t, uc);
    else if (kern_s) kern_s<<<(unsigned)grid, MS_BLOCK, 0, st>>>(pc, t, u);
    else kern<<<(unsigned)grid, MS_BLOCK, 0, st>>>(p, t, MsNoSum{});
    CUDA_TRY(cudaGetLastError());
    g_launches++;
    return PFW_OK;
}

int launch_ms(pfw_ruleset *h, int mode, const ScanParams &p, cudaStream_t st) {
    switch (mode) {
        case MODE_ACC: return launch_ms_k<MODE_ACC>(h, p, st);
        case MODE_PEER: return launch_ms_k<MODE_PEER>(h, p, st);
        default: return launch_ms_k<MODE_WRITE>(h, p, st);
    }
}

