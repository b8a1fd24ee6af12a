/*
 * pfw.h -- C-ABI of the B200 packet-filter hot path (libpfw.so).
 *
 * The reference (parafw, pure Python) has no FFI; these entry points are the
 * functions its classify path would bind if its numpy inner loop were moved
 * behind a native library.  Each one names the reference interface it
 * replaces (/root/reference/pkg/src/parafw/<file>:<line>).
 * shows the ctypes binding a parafw maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only; no exceptions cross the ABI.  Every call
 *    returns PFW_OK (0) or a PFW_ERR_* code; pfw_last_error() describes the
 *    last failure on the calling thread.
 *  - "d_" pointers are device pointers on the ruleset's device, "h_" pointers
 *    are host pointers (pinned memory gives overlapped copies).
 *  - stream arguments are cudaStream_t passed as void* (NULL = legacy stream).
 *  - Device calls are asynchronous on the stream unless stated otherwise.
 *  - Packets are 16-byte records: {src_ip, dst_ip, (src_port<<16)|dst_port,
 *    proto} (uint32 x4), the packet-batch layout that replaces the 5-column
 *    PacketArrays (classifier.py:62-95).
 *  - A first-match index is a uint32 global rule index; PFW_NO_MATCH means no
 *    rule in the scanned window matched (the reference's -1, default deny).
 *    PFW_NO_MATCH is INT32_MAX so that it is also the identity of an int32 or
 *    uint32 MIN reduction (the function-parallel combine).
 *  - A handle is bound to one device and is not reentrant (mirrors Engine,
 *    engines.py:221-228); different handles may be driven concurrently.
 */
#ifndef PFW_H
#define PFW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFW_NO_MATCH 0x7FFFFFFFu
/* pfw_classify_host_ex flags */
#define PFW_HOST_FIRST_MINUS1 1u /* unmatched packets get first = 0xFFFFFFFF (int32 -1, scan_range's value) */
#define PFW_MAX_RULES 0x7FFFFFFE

enum {
    PFW_OK = 0,
    PFW_ERR_INVALID = 1, /* bad argument (the reference's ValueError / ConfigError) */
    PFW_ERR_CUDA = 2,    /* CUDA runtime failure */
    PFW_ERR_NOMEM = 3,   /* device or host allocation failure */
    PFW_ERR_GENERATION = 4 /* traffic generation failed */
};

typedef struct pfw_ruleset *pfw_ruleset_t;

/* Description of the last failure on this thread ("" if none). */
const char *pfw_last_error(void);

/* Library / build information: "pfw <version> sm_100a ...". */
const char *pfw_version(void);

/* Number of visible CUDA devices (0 when no GPU); never fails. */
int pfw_device_count(void);

/* Ruleset packing + upload.  Replaces CompiledRuleset.__init__
 * (classifier.py:120-134): takes exactly its ten SoA columns (proto u8 with
 * ANY = 0, CIDR base/mask u32, inclusive port lo/hi u16, action_accept u8)
 * and uploads the device forms once: the range-test SoA of the rule-by-rule
 * scan and, within the memory budget, the per-field match sets (interval
 * bitmaps).  Rules whose base has host bits outside the mask, or
 * whose port range is inverted, can never match under the reference
 * predicate (model.py:222-230) and are packed as never-matching.  Masks must
 * be CIDR prefix masks (model.py:108-114; anything else is PFW_ERR_INVALID).
 * n_rules may be 0. */
int pfw_ruleset_create(int device, int64_t n_rules, const uint8_t *proto,
                       const uint32_t *src_base, const uint32_t *src_mask,
                       const uint16_t *sport_lo, const uint16_t *sport_hi,
                       const uint32_t *dst_base, const uint32_t *dst_mask,
                       const uint16_t *dport_lo, const uint16_t *dport_hi,
                       const uint8_t *action_accept, pfw_ruleset_t *out);
int pfw_ruleset_destroy(pfw_ruleset_t h);
int64_t pfw_ruleset_size(pfw_ruleset_t h);
int pfw_ruleset_device(pfw_ruleset_t h);
/* Device bytes of the ruleset's match sets; 0 when they were not built (the
 * ruleset then scans rule by rule). */
int64_t pfw_ruleset_matchset_bytes(pfw_ruleset_t h);
/* Mark the handle as a rule shard: its rules are positions [index_base,
 * index_base + n) of an ordered ruleset of `total` rules (function-parallel:
 * each GPU uploads only its partition, engines.py:316-321).  Scan windows stay
 * in local positions [0, n); every reported first-match index (outputs, the
 * accumulate min, the fused peer combine) becomes index_base + local; the
 * comparison counts are window-relative as before.  pfw_verdicts rejects a
 * partial shard (combined indices need the whole ruleset's actions). */
int pfw_ruleset_set_shard(pfw_ruleset_t h, int64_t index_base, int64_t total);
/* Ruleset introspection: "matchset_bytes", "compressed" (1: compressed match-set
 * rows), "summaries" (1: the scan uses block summaries), "index_base". */
int pfw_ruleset_info(pfw_ruleset_t h, const char *key, int64_t *value);

/* Host packet packing.  Replaces PacketArrays.from_packets
 * (classifier.py:75-83) for column input: writes n 16-byte records. */
int pfw_pack_packets_host(int64_t n, const uint8_t *proto, const uint32_t *src_ip,
                          const uint16_t *src_port, const uint32_t *dst_ip,
                          const uint16_t *dst_port, void *h_out);

/* First-match scan over the rule window [lo, hi).  Replaces
 * CompiledRuleset.scan_range (classifier.py:146-162) and the sequential /
 * data-parallel comparison accounting (classifier.py:200, engines.py:312):
 *   d_first[i]   = earliest matching global rule index in [lo, hi) or
 *                  PFW_NO_MATCH (lo >= hi or n == 0: all PFW_NO_MATCH / no-op)
 *   d_comps[i]   = first - lo + 1, or hi - lo on a miss     (nullable)
 *   d_verdict[i] = 1 iff a rule matched and it is ACCEPT    (nullable)
 *   d_stats[0] += sum of comps, d_stats[1] = max(d_stats[1], max comps)
 *                                                            (nullable) */
int pfw_scan_range(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts, int64_t n,
                   uint32_t *d_first, uint32_t *d_comps, uint8_t *d_verdict,
                   uint64_t *d_stats, void *stream);

/* Same scan reading the reference's own column layout (PacketArrays,
 * classifier.py:62-95: proto u8, src_ip u32, src_port u16, dst_ip u32,
 * dst_port u16 -- 13 bytes per packet) directly, no packing step. */
int pfw_scan_range_columns(pfw_ruleset_t h, int64_t lo, int64_t hi, const uint8_t *d_proto,
                           const uint32_t *d_src_ip, const uint16_t *d_src_port, const uint32_t *d_dst_ip,
                           const uint16_t *d_dst_port, int64_t n, uint32_t *d_first, uint32_t *d_comps,
                           uint8_t *d_verdict, uint64_t *d_stats, void *stream);

/* One partition of the function-parallel / hybrid models.  Replaces a
 * _scan_partitions task + its share of _combine_rows (engines.py:349-369):
 *   d_first[i]  = min(d_first[i], partition-local first match)
 *   d_comps[i] += per-task comparisons (local - lo + 1, or hi - lo)
 *   d_stats[0] += sum of per-task comparisons, d_stats[1] = max(..., per-task)
 * d_first must start at PFW_NO_MATCH and d_comps at 0 (pfw_accumulator_init). */
int pfw_scan_partition_accumulate(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts,
                                  int64_t n, uint32_t *d_first, uint32_t *d_comps,
                                  uint64_t *d_stats, void *stream);
int pfw_accumulator_init(int64_t n, uint32_t *d_first, uint32_t *d_comps, void *stream);

/* Every node of the function-parallel / hybrid models on one device
 * (engines.py:349-369 over partition_bounds(R, nodes), engines.py:140-154):
 *   d_first[i] = the lowest node's local first match (PFW_NO_MATCH: none)
 *   d_comps[i] = the sum over nodes of local - lo + 1, or hi - lo
 *   d_stats[0] += sum of d_comps, d_stats[1] = max(..., largest per-node count)
 * Runs pfw_accumulator_init + pfw_scan_partition_accumulate over each
 * non-empty partition on the stream.  Overwrites d_first / d_comps; d_stats
 * may be NULL.  Replaces the per-node loop of
 * engines.py:349-369 (FUNCTION_PARALLEL / HYBRID with nodes partitions). */
int pfw_scan_partitions(pfw_ruleset_t h, int64_t nodes, const void *d_pkts, int64_t n, uint32_t *d_first,
                        uint32_t *d_comps, uint64_t *d_stats, void *stream);

/* Fused function-parallel combine.  Scans the rule shard
 * [lo, hi) like pfw_scan_partition_accumulate, but the kernel epilogue folds
 * each resolved packet straight into the ranks' result buffers with NVLink
 * atomics (atomicMin of the first match, atomicAdd of the per-task
 * comparisons), replacing the separate NCCL MIN all-reduce of
 * engines.py:202-212 and the sum of engines.py:366-367.
 *   h_peer_first[t] / h_peer_comps[t]: rank t's buffers as mapped in this
 *     process (pfw_ipc_open; the caller's own buffer for its own rank);
 *     h_peer_comps may be NULL.  Buffers start at PFW_NO_MATCH / 0.
 *   h_peer_cap[t]: packets rank t's buffers hold; a call whose n needs more
 *     (its shard of n, or n) fails with PFW_ERR_INVALID before any launch.
 *   scatter = 0: every rank's buffer holds all n packets (all-reduce result);
 *   scatter = 1: packet i is held by its owner rank (balanced contiguous
 *     shards of n, partition_bounds semantics) at offset i - shard start
 *     (reduce-scatter result, one atomic per packet).
 * Completion: the combine is complete on every rank once all ranks' kernels
 * have finished (e.g. stream synchronize + a host barrier). */
int pfw_scan_fused_min(pfw_ruleset_t h, int64_t lo, int64_t hi, const void *d_pkts, int64_t n,
                       uint32_t *const *h_peer_first, uint32_t *const *h_peer_comps,
                       const int64_t *h_peer_cap, int npeers, int scatter, uint64_t *d_stats, void *stream);

/* In-process multi-GPU fused combine (Engine(devices=...)): let `device`'s
 * kernels access `peer`'s memory directly over NVLink (cudaDeviceEnablePeerAccess);
 * already enabled, or device == peer, is success. */
int pfw_peer_enable(int device, int peer);

/* CUDA IPC plumbing for the fused combine.  pfw_ipc_get_handle exports the
 * allocation containing d_ptr and returns d_ptr's byte offset in it;
 * pfw_ipc_open maps a peer's allocation (NVLink peer access) and returns its
 * BASE -- add the exported offset; pfw_ipc_close unmaps that base. */
int pfw_ipc_handle_size(void);
int pfw_ipc_get_handle(const void *d_ptr, void *out_handle, uint64_t *offset);
int pfw_ipc_open(int device, const void *handle, void **out_base);
int pfw_ipc_close(int device, void *base);

/* Verdicts from final first-match indices (classifier.py:175-185). */
int pfw_verdicts(pfw_ruleset_t h, const uint32_t *d_first, int64_t n, uint8_t *d_verdict,
                 void *stream);

/* Per-packet minimum over partitions (engines.py:202-212) for W rows of n
 * indices laid out row-major: d_out[i] = min_w d_rows[w*n + i]. */
int pfw_combine_min(const uint32_t *d_rows, int64_t rows, int64_t n, uint32_t *d_out, void *stream);

/* End-to-end sequential classification with HOST buffers.  Replaces
 * classify_batch_sequential (classifier.py:192-209) minus object building:
 * copies packets in `chunk`-packet pieces to the device, scans [0, R) and
 * copies first-match indices / verdicts back, overlapping copies with the
 * kernels on two streams.  Synchronous: all outputs are complete on return.
 * h_verdict and h_stats ([sum, max] comparisons) are nullable. */
int pfw_classify_host(pfw_ruleset_t h, const void *h_pkts, int64_t n, uint32_t *h_first,
                      uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk);

/* pfw_classify_host for the reference's column layout (PacketArrays):
 * copies 13 bytes per packet (five column copies per chunk), no host packing.
 * Both host entry points take pinned or pageable buffers: pageable ones are
 * staged through a per-handle pinned ring by a host thread pool, chunk by
 * chunk, overlapping the device copies and scans. */
int pfw_classify_host_columns(pfw_ruleset_t h, const uint8_t *h_proto, const uint32_t *h_src_ip,
                              const uint16_t *h_src_port, const uint32_t *h_dst_ip,
                              const uint16_t *h_dst_port, int64_t n, uint32_t *h_first,
                              uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk);

/* Either entry point with flags: h_pkts (16-byte records) non-NULL selects
 * the record layout, otherwise the five columns are read.  flags:
 * PFW_HOST_FIRST_MINUS1 writes -1 for unmatched packets, so h_first is the
 * reference's scan_range result (classifier.py:146-162) as int32. */
int pfw_classify_host_ex(pfw_ruleset_t h, const void *h_pkts, const uint8_t *h_proto,
                         const uint32_t *h_src_ip, const uint16_t *h_src_port, const uint32_t *h_dst_ip,
                         const uint16_t *h_dst_port, int64_t n, uint32_t *h_first, uint8_t *h_verdict,
                         uint64_t *h_stats, int64_t chunk, uint32_t flags);

/* The same pipeline for the function-parallel / hybrid models (engines.py:
 * 316-369 over partition_bounds(R, nodes)): each chunk runs every node's
 * partition scan folded on the device (pfw_scan_partitions), so h_first =
 * the lowest node's match, h_comps = the per-packet sum over nodes of the
 * per-task comparisons, h_stats = [sum, largest per-node count]; verdicts
 * from h_first.  Whole rulesets only (not a rule shard).  h_comps required. */
int pfw_classify_host_partitions(pfw_ruleset_t h, int64_t nodes, const void *h_pkts, const uint8_t *h_proto,
                                 const uint32_t *h_src_ip, const uint16_t *h_src_port, const uint32_t *h_dst_ip,
                                 const uint16_t *h_dst_port, int64_t n, uint32_t *h_first, uint32_t *h_comps,
                                 uint8_t *h_verdict, uint64_t *h_stats, int64_t chunk, uint32_t flags);

/* Bit-exact UNIFORM traffic generation on the device.  Replaces
 * generate_traffic(TrafficProfile(...)) with match_mode UNIFORM
 * (traffic.py:117-130, 148-160; rng.py:31-62): the pinned xorshift64* stream
 * is split across threads by GF(2) jump-ahead.  Synchronous (it checks for
 * the rare bounded-draw rejection and repairs the stream exactly).  Writes n
 * packed packets to d_out. */
int pfw_generate_traffic(int device, uint64_t seed, int64_t n, int proto, uint32_t src_base,
                         int src_plen, uint32_t dst_base, int dst_plen, int sport_lo,
                         int sport_hi, int dport_lo, int dport_hi, void *d_out, void *stream);

/* Same stream, packets [first_packet, first_packet + n) only (one rank's
 * shard of a global batch, engines.py:307 / partition_bounds).  first_packet
 * > 0 requires power-of-two port spans, where every packet is exactly four
 * draws; the default wildcard profile qualifies. */
int pfw_generate_traffic_at(int device, uint64_t seed, int64_t first_packet, int64_t n, int proto,
                            uint32_t src_base, int src_plen, uint32_t dst_base, int dst_plen,
                            int sport_lo, int sport_hi, int dport_lo, int dport_hi, void *d_out,
                            void *stream);

/* Native readers / writers of the formats feeding the path (hostio.cpp).
 * They accept the canonical grammar strictly and return PFW_ERR_INVALID with
 * pfw_io_last_error() = "line N: ..." at the first line they cannot accept;
 * callers then re-read with the reference-compatible parser (exact errors).
 *   pfw_parse_rules    ruleset text (model.py:7-20, 233-331) -> the ten
 *                      CompiledRuleset columns (classifier.py:120-134)
 *   pfw_parse_traffic  traffic CSV (traffic.py:259-297) -> ids + 16-byte records
 *   pfw_format_results "id,VERDICT,index|-" lines (cli.py:62-65) */
const char *pfw_io_last_error(void);
int pfw_parse_rules(const char *buf, int64_t len, int64_t cap, uint8_t *proto, uint32_t *src_base,
                    uint32_t *src_mask, uint16_t *sport_lo, uint16_t *sport_hi, uint32_t *dst_base,
                    uint32_t *dst_mask, uint16_t *dport_lo, uint16_t *dport_hi, uint8_t *accept,
                    int64_t *n_out);
int pfw_parse_traffic(const char *buf, int64_t len, int64_t cap, int64_t *ids, void *h_records,
                      int64_t *n_out);
int pfw_format_results(const int64_t *ids, const uint32_t *first, const uint8_t *verdict, int64_t n,
                       char *out, int64_t cap, int64_t *written);

/* Launch-count / tuning introspection (bench + tests).  Tuning values are
 * process-wide and not synchronised: set them before issuing scans from
 * several host threads.  Results never depend on them.  Tuning keys include
 * "algo" (0 auto: match sets when built, 1 rule-by-rule scan, 2 match sets),
 * "matchset" (build match sets at ruleset creation, default 1),
 * "matchset_budget_mb" (0 = a quarter of free device memory), "ms_compress"
 * (compressed rows: 0 off, 1 on, 2 auto), "ms_group"
 * (lanes per packet), "ms_words" (words per lane per step), "ms_summary" (1024-rule
 * block summaries: 0 off, 1 on, 2 auto; applies to rulesets created afterwards),
 * and the rule-scan options "ks", "tile", "first_pass", "bucket",
 * "bucket_min", "proto_split", "short_circuit", "force_imad", "ctas_per_sm". */
int64_t pfw_launch_count(void);
/* L2 read-bandwidth probe (bench.py's roofline peak, measured live): on the
 * current device, blocks_per_sm x SMs blocks of 256 threads, each group of 8
 * lanes reading one random 128-byte line of d_buf (>= 1 MiB, L2-resident
 * size) per load, lines_in_flight (2, 4, 8 or 16) per lane per iteration, iters
 * iterations; bytes read = SMs x blocks_per_sm x 32 x lines_in_flight x iters
 * x 128.  The caller times it (events on the stream). */
int pfw_probe_l2_lines(const void *d_buf, int64_t bytes, int lines_in_flight, int blocks_per_sm, int iters,
                       void *stream);
/* Instrumentation counters, read and reset: "blocks_read" = 1024-rule blocks
 * the match-set scan with block summaries read (counted while tuning
 * "count_blocks" is 1; used by bench.py for that variant's roofline). */
int pfw_read_counter(const char *name, int64_t *value);
int pfw_set_tuning(const char *key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* PFW_H */
