// hostio.cpp -- native readers/writers for the formats that feed the hot path
// (SURVEY 8(f) row 4 / row 2):
//   ruleset text   model.py:7-20, 233-331   -> CompiledRuleset columns
//   traffic CSV    traffic.py:12-13, 259-297 -> 16-byte packet records + ids
//   results        cli.py:62-65             -> "id,VERDICT,index|-" lines
//
// The parsers accept the canonical grammar strictly.  They return
// PFW_ERR_INVALID with the 1-based line number of the first line they cannot
// accept; the Python layer then re-reads the file with the reference-
// compatible parser, which yields either the reference's exact error or the
// value of a non-canonical-but-valid spelling (e.g. "+80").  Well-formed
// files never leave the native path.
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <string>

#include "../../include/pfw.h"

namespace {

thread_local std::string g_io_err;

int io_err(int64_t line, const char *what) {
    char buf[256];
    snprintf(buf, sizeof buf, "line %lld: %s", (long long)line, what);
    g_io_err = buf;
    return PFW_ERR_INVALID;
}

struct Cursor {
    const char *p, *end;
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\f' || c == '\v'; }

// next whitespace-separated token inside [p, end); false at end
inline bool token(Cursor &c, const char *&t0, const char *&t1) {
    while (c.p < c.end && is_space(*c.p)) c.p++;
    if (c.p >= c.end) return false;
    t0 = c.p;
    while (c.p < c.end && !is_space(*c.p)) c.p++;
    t1 = c.p;
    return true;
}

inline bool eq(const char *a, const char *b, const char *lit) {
    const size_t n = strlen(lit);
    return (size_t)(b - a) == n && memcmp(a, lit, n) == 0;
}

// canonical unsigned decimal: [0-9]+, no sign, value <= max (leading zeros ok,
// as Python int() accepts them)
inline bool parse_uint(const char *a, const char *b, uint64_t max, uint64_t &out) {
    if (a >= b || b - a > 19) return false;
    uint64_t v = 0;
    for (const char *q = a; q < b; q++) {
        if (*q < '0' || *q > '9') return false;
        v = v * 10 + (uint64_t)(*q - '0');
    }
    if (v > max) return false;
    out = v;
    return true;
}

// dotted quad as ipaddress.IPv4Address accepts it: 4 decimal octets 0..255,
// 1-3 digits, no leading zeros (except "0")
inline bool parse_ip(const char *a, const char *b, uint32_t &out) {
    uint32_t v = 0;
    int parts = 0;
    const char *q = a;
    while (parts < 4) {
        const char *s = q;
        while (q < b && *q >= '0' && *q <= '9') q++;
        const long n = q - s;
        if (n < 1 || n > 3) return false;
        if (n > 1 && *s == '0') return false;
        uint64_t o;
        if (!parse_uint(s, q, 255, o)) return false;
        v = (v << 8) | (uint32_t)o;
        parts++;
        if (parts < 4) {
            if (q >= b || *q != '.') return false;
            q++;
        }
    }
    if (q != b) return false;
    out = v;
    return true;
}

inline bool parse_cidr(const char *a, const char *b, uint32_t &base, uint32_t &mask) {
    if (eq(a, b, "*")) {
        base = mask = 0;
        return true;
    }
    const char *slash = (const char *)memchr(a, '/', (size_t)(b - a));
    if (!slash) return false;
    uint32_t ip;
    uint64_t plen;
    if (!parse_ip(a, slash, ip) || !parse_uint(slash + 1, b, 32, plen)) return false;
    mask = plen == 0 ? 0u : (uint32_t)(0xFFFFFFFFull << (32 - plen));  // model.py:108-114
    base = ip & mask;                                                   // model.py:106
    return true;
}

inline bool parse_ports(const char *a, const char *b, uint16_t &lo, uint16_t &hi) {
    if (eq(a, b, "*")) {
        lo = 0;
        hi = 65535;
        return true;
    }
    const char *dash = (const char *)memchr(a, '-', (size_t)(b - a));
    uint64_t l, h;
    if (!dash) {
        if (!parse_uint(a, b, 65535, l)) return false;
        h = l;
    } else if (!parse_uint(a, dash, 65535, l) || !parse_uint(dash + 1, b, 65535, h)) {
        return false;
    }
    if (l > h) return false;  // inverted range: the Python path raises the exact error
    lo = (uint16_t)l;
    hi = (uint16_t)h;
    return true;
}

inline int proto_code(const char *a, const char *b, bool allow_any) {
    if (eq(a, b, "tcp")) return 6;
    if (eq(a, b, "udp")) return 17;
    if (eq(a, b, "icmp")) return 1;
    if (allow_any && eq(a, b, "any")) return 0;
    return -1;
}

}  // namespace

extern "C" {

const char *pfw_io_last_error(void) { return g_io_err.c_str(); }

int pfw_parse_rules(const char *buf, int64_t len, int64_t cap, uint8_t *proto, uint32_t *src_base,
                    uint32_t *src_mask, uint16_t *sport_lo, uint16_t *sport_hi, uint32_t *dst_base,
                    uint32_t *dst_mask, uint16_t *dport_lo, uint16_t *dport_hi, uint8_t *accept,
                    int64_t *n_out) {
    if (!buf || len < 0 || !n_out) return io_err(0, "bad arguments");
    int64_t n = 0, line = 0;
    const char *p = buf, *end = buf + len;
    while (p < end) {
        const char *eol = (const char *)memchr(p, '\n', (size_t)(end - p));
        if (!eol) eol = end;
        line++;
        const char *hash = (const char *)memchr(p, '#', (size_t)(eol - p));  // model.py:314-316
        Cursor c{p, hash ? hash : eol};
        p = eol + 1;
        const char *t[6][2];
        int k = 0;
        while (k < 6 && token(c, t[k][0], t[k][1])) k++;
        if (k == 0) continue;  // blank / comment-only line
        const char *x0, *x1;
        if (k < 6 || token(c, x0, x1)) return io_err(line, "expected 6 fields");
        if (n >= cap) return io_err(line, "capacity exceeded");
        int act;
        if (eq(t[0][0], t[0][1], "ACCEPT")) act = 1;
        else if (eq(t[0][0], t[0][1], "DROP")) act = 0;
        else return io_err(line, "field 1");
        const int pr = proto_code(t[1][0], t[1][1], true);
        if (pr < 0) return io_err(line, "field 2");
        if (!parse_cidr(t[2][0], t[2][1], src_base[n], src_mask[n])) return io_err(line, "field 3");
        if (!parse_ports(t[3][0], t[3][1], sport_lo[n], sport_hi[n])) return io_err(line, "field 4");
        if (!parse_cidr(t[4][0], t[4][1], dst_base[n], dst_mask[n])) return io_err(line, "field 5");
        if (!parse_ports(t[5][0], t[5][1], dport_lo[n], dport_hi[n])) return io_err(line, "field 6");
        proto[n] = (uint8_t)pr;
        accept[n] = (uint8_t)act;
        n++;
    }
    *n_out = n;
    return PFW_OK;
}

int pfw_parse_traffic(const char *buf, int64_t len, int64_t cap, int64_t *ids, void *records,
                      int64_t *n_out) {
    if (!buf || len < 0 || !n_out) return io_err(0, "bad arguments");
    static const char header[] = "id,proto,src_ip,src_port,dst_ip,dst_port";  // traffic.py:55
    const char *p = buf, *end = buf + len;
    const char *eol = (const char *)memchr(p, '\n', (size_t)(end - p));
    if (!eol) eol = end;
    const char *he = (eol > p && eol[-1] == '\r') ? eol - 1 : eol;
    if (!eq(p, he, header)) return io_err(1, "header");
    p = eol < end ? eol + 1 : end;
    uint32_t *rec = static_cast<uint32_t *>(records);
    int64_t n = 0, line = 1;
    while (p < end) {
        eol = (const char *)memchr(p, '\n', (size_t)(end - p));
        if (!eol) eol = end;
        line++;
        const char *le = (eol > p && eol[-1] == '\r') ? eol - 1 : eol;
        const char *q = p;
        p = eol + 1;
        if (q == le) continue;  // empty row (traffic.py:270-271)
        const char *f[6][2];
        int k = 0;
        while (k < 6) {
            const char *s = q;
            while (q < le && *q != ',') q++;
            f[k][0] = s;
            f[k][1] = q;
            k++;
            if (q >= le) break;
            q++;
        }
        if (k != 6 || q < le) return io_err(line, "expected 6 columns");
        if (n >= cap) return io_err(line, "capacity exceeded");
        uint64_t id, sp, dp;
        uint32_t src, dst;
        // ids: canonical non-negative decimal (other int() spellings -> Python path)
        if (!parse_uint(f[0][0], f[0][1], (uint64_t)INT64_MAX, id)) return io_err(line, "id");
        const int pr = proto_code(f[1][0], f[1][1], false);
        if (pr < 0) return io_err(line, "protocol");
        if (!parse_ip(f[2][0], f[2][1], src) || !parse_ip(f[4][0], f[4][1], dst)) return io_err(line, "ip");
        if (!parse_uint(f[3][0], f[3][1], 65535, sp) || !parse_uint(f[5][0], f[5][1], 65535, dp))
            return io_err(line, "port");
        ids[n] = (int64_t)id;
        rec[4 * n + 0] = src;
        rec[4 * n + 1] = dst;
        rec[4 * n + 2] = ((uint32_t)sp << 16) | (uint32_t)dp;
        rec[4 * n + 3] = (uint32_t)pr;
        n++;
    }
    *n_out = n;
    return PFW_OK;
}

int pfw_format_results(const int64_t *ids, const uint32_t *first, const uint8_t *verdict, int64_t n,
                       char *out, int64_t cap, int64_t *written) {
    if (n < 0 || !written || (n > 0 && (!ids || !first || !verdict || !out)))
        return io_err(0, "bad arguments");
    char *o = out, *oe = out + cap;
    for (int64_t i = 0; i < n; i++) {
        if (oe - o < 48) return io_err(i, "output buffer too small");
        o += snprintf(o, (size_t)(oe - o), "%lld,", (long long)ids[i]);
        const char *v = verdict[i] ? "ACCEPT" : "DROP";
        const size_t vl = verdict[i] ? 6 : 4;
        memcpy(o, v, vl);
        o += vl;
        *o++ = ',';
        if (first[i] == PFW_NO_MATCH) {
            *o++ = '-';
        } else {
            o += snprintf(o, (size_t)(oe - o), "%u", first[i]);
        }
        *o++ = '\n';
    }
    *written = o - out;
    return PFW_OK;
}

}  // extern "C"
