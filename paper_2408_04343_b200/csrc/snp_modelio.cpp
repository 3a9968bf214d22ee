// snp_modelio.cpp -- native model-file parser and writer (include/snpio.h).
//
// Same grammar, checks, check order and messages as the reference's
// parse_model / serialize_model (pkg/src/snpsim/modelfile.py:40-143) and the
// builder invariants it triggers (model.py:50-112 SpikeRegex/Rule,
// model.py:155-180 add_neuron/add_rule/add_synapse), but single pass over a
// byte buffer into flat arrays: rules are regrouped by owner with a stable
// counting pass (validate(), model.py:251) and synapses become a sorted,
// de-duplicated CSR (model.py:255-257).
//
// Deviations (documented in DESIGN.md): integers must fit int64 (the
// reference's Python ints are unbounded; larger values would fail the
// engine's int32/int64 range checks anyway), neuron counts must be < 2^32,
// and only ASCII line breaks / whitespace are recognised.
#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/snpio.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// Python repr() of a str made of the given bytes (ASCII escapes; other
// bytes pass through as UTF-8).
std::string py_repr(const char* p, size_t n) {
    bool has_sq = memchr(p, '\'', n) != nullptr, has_dq = memchr(p, '"', n) != nullptr;
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string s(1, q);
    for (size_t i = 0; i < n; ++i) {
        const unsigned char c = (unsigned char)p[i];
        if (c == '\\') s += "\\\\";
        else if (c == (unsigned char)q) { s += '\\'; s += (char)c; }
        else if (c == '\t') s += "\\t";
        else if (c == '\n') s += "\\n";
        else if (c == '\r') s += "\\r";
        else if (c < 0x20 || c == 0x7f) {
            char b[8];
            snprintf(b, sizeof(b), "\\x%02x", c);
            s += b;
        } else s += (char)c;
    }
    s += q;
    return s;
}

inline bool is_break(unsigned char c) { return c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1e); }
inline bool is_space(unsigned char c) { return c == ' ' || c == '\t' || is_break(c) || c == 0x1f; }

struct Tok {
    const char* p;
    size_t n;
    bool is(const char* s) const { return strlen(s) == n && memcmp(p, s, n) == 0; }
    std::string repr() const { return py_repr(p, n); }
};

// int(token) as Python parses it: optional sign, digits with single
// underscores between them.  0 ok, 1 not an integer, 2 outside int64.
int parse_int(const Tok& t, long long* out) {
    size_t i = 0;
    bool neg = false;
    if (i < t.n && (t.p[i] == '+' || t.p[i] == '-')) neg = t.p[i++] == '-';
    if (i >= t.n) return 1;
    unsigned long long v = 0;
    bool over = false, prev_digit = false;
    for (; i < t.n; ++i) {
        const char c = t.p[i];
        if (c == '_') {
            if (!prev_digit || i + 1 >= t.n) return 1;
            prev_digit = false;
            continue;
        }
        if (c < '0' || c > '9') return 1;
        prev_digit = true;
        if (v > (~0ull - 9) / 10) over = true;
        v = v * 10 + (unsigned long long)(c - '0');
        if (v > (1ull << 63)) over = true;
    }
    if (!prev_digit) return 1;
    if (over || (!neg && v > (unsigned long long)INT64_MAX)) return 2;
    *out = neg ? (long long)(0ull - v) : (long long)v;
    return 0;
}

}  // namespace

struct snpio_model {
    std::vector<long long> initial;
    // rules in file order (regrouped by owner in export)
    std::vector<uint32_t> owner;
    std::vector<long long> thr, cons, prod, dly;
    std::vector<uint8_t> exact;
    std::vector<unsigned long long> syn;  // src << 32 | dst, file order (duplicates allowed)
    long long output = -1;
    // CSR built at the end of parsing
    std::vector<long long> adj_off, adj_dst;
};

namespace {

// f(i, thread) for i in [0, n) over up to `threads` threads (contiguous ranges).
template <class F>
void for_each_index(size_t n, size_t threads, F&& f) {
    threads = std::max<size_t>(1, std::min(threads, n));
    if (threads == 1) {
        for (size_t i = 0; i < n; ++i) f(i, 0);
        return;
    }
    std::vector<std::thread> th;
    for (size_t t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
            for (size_t i = n * t / threads, e = n * (t + 1) / threads; i < e; ++i) f(i, t);
        });
    for (auto& x : th) x.join();
}

// Parsed output of one text range (the whole file, or one chunk of it).
struct Sink {
    std::vector<long long> initial;
    std::vector<uint32_t> owner;
    std::vector<long long> thr, cons, prod, dly;
    std::vector<uint8_t> exact;
    std::vector<unsigned long long> syn;
    long long output = -1;
};

struct Parser {
    snpio_model* m = nullptr;
    Sink* out = nullptr;        // where rules / synapses / output go
    long long lineno = 0;
    bool header = false, spikes = false;
    long long count = -1;
    int err_code = SNPIO_OK;
    std::string err;            // message of the first error (thread-local parsing)
    std::vector<Tok> args;

    int efail(int code, const char* fmt, ...) {
        char buf[1024];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        err = buf;
        err_code = code;
        return code;
    }
    int ferr(const char* fmt, ...) {
        char buf[900];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        return efail(SNPIO_ERR_FORMAT, "line %lld: %s", lineno, buf);
    }
    // modelfile.py:151-160
    int get_int(size_t pos, const char* what, long long* v) {
        if (pos >= args.size()) return ferr("missing %s", what);
        const int rc = parse_int(args[pos], v);
        if (rc == 1) return ferr("%s must be an integer, got %s", what, args[pos].repr().c_str());
        if (rc == 2) return ferr("%s out of range for the native parser, got %s", what, args[pos].repr().c_str());
        return SNPIO_OK;
    }
    // modelfile.py:163-167
    int get_index(size_t pos, long long cnt, long long* v) {
        long long x;
        if (int rc = get_int(pos, "neuron index", &x)) return rc;
        if (x < 1 || x > cnt) return ferr("neuron index %lld out of range 1..%lld", x, cnt);
        *v = x - 1;
        return SNPIO_OK;
    }

    // One line of modelfile.py:74-135 (raw excludes the line break).
    int line(const char* raw, size_t raw_n) {
        ++lineno;
        const char* hash = (const char*)memchr(raw, '#', raw_n);
        const size_t n = hash ? (size_t)(hash - raw) : raw_n;
        args.clear();
        for (size_t k = 0; k < n;) {
            while (k < n && is_space((unsigned char)raw[k])) ++k;
            size_t b = k;
            while (k < n && !is_space((unsigned char)raw[k])) ++k;
            if (k > b) args.push_back(Tok{raw + b, k - b});
        }
        if (args.empty()) return SNPIO_OK;
        const Tok key = args.front();
        args.erase(args.begin());
        if (!header) {
            if (!key.is("snp")) return ferr("expected 'snp <version>' header, got %s", py_repr(raw, raw_n).c_str());
            long long ver;
            if (int rc = get_int(0, "format version", &ver)) return rc;
            if (ver != 1) return ferr("unsupported format version %lld", ver);
            header = true;
        } else if (key.is("neurons")) {
            if (count >= 0) return ferr("duplicate 'neurons' line");
            if (int rc = get_int(0, "neuron count", &count)) return rc;
            if (count < 0) return ferr("neuron count must be >= 0");
            if (count >= (1ll << 32) - 1) return ferr("neuron count %lld too large for the native parser", count);
        } else if (key.is("spikes")) {
            if (count < 0) return ferr("'spikes' before 'neurons'");
            if (spikes) return ferr("duplicate 'spikes' line");
            if ((long long)args.size() != count) return ferr("expected %lld spike counts, got %zu", count, args.size());
            out->initial.reserve((size_t)count);
            for (long long p = 0; p < count; ++p) {
                long long v;
                if (int rc = get_int((size_t)p, "spike count", &v)) return rc;
                if (v < 0) return efail(SNPIO_ERR_MODEL, "initial spike count must be >= 0, got %lld", v);
                out->initial.push_back(v);
            }
            spikes = true;
        } else if (key.is("rule") || key.is("synapse") || key.is("output")) {
            if (!spikes) return ferr("directive before 'spikes' line");
            if (key.is("rule")) {
                if (args.size() != 6) return ferr("'rule' needs 6 fields, got %zu", args.size());
                int exact;
                if (args[1].is("ge")) exact = 0;
                else if (args[1].is("eq")) exact = 1;
                else return ferr("condition kind must be 'ge' or 'eq', got %s", args[1].repr().c_str());
                long long own = 0, t = 0, c = 0, p = 0, d = 0;
                if (int rc = get_index(0, count, &own)) return rc;
                if (int rc = get_int(2, "threshold", &t)) return rc;
                // SpikeRegex (model.py:50-55)
                if (t < 0) return efail(SNPIO_ERR_INVALID_RULE, "condition threshold must be >= 0, got %lld", t);
                if (exact && t < 1) return efail(SNPIO_ERR_INVALID_RULE, "an exact-count condition needs threshold >= 1");
                if (int rc = get_int(3, "consumed", &c)) return rc;
                if (int rc = get_int(4, "produced", &p)) return rc;
                if (int rc = get_int(5, "delay", &d)) return rc;
                // Rule (model.py:87-106)
                if (c < 1) return efail(SNPIO_ERR_INVALID_RULE, "a rule must consume at least one spike, got %lld", c);
                if (p < 0) return efail(SNPIO_ERR_INVALID_RULE, "produced spike count must be >= 0, got %lld", p);
                if (d < 0) return efail(SNPIO_ERR_INVALID_RULE, "delay must be >= 0, got %lld", d);
                if (p == 0) {
                    if (d != 0) return efail(SNPIO_ERR_INVALID_RULE, "a forgetting rule cannot carry a delay");
                    if (!exact || t != c)
                        return efail(SNPIO_ERR_INVALID_RULE, "a forgetting rule must be guarded by exactly its consumed count");
                } else if (p > c) {
                    return efail(SNPIO_ERR_INVALID_RULE,
                                 "a firing rule cannot produce more than it consumes (consumed=%lld, produced=%lld)", c, p);
                }
                out->owner.push_back((uint32_t)own);
                out->thr.push_back(t);
                out->exact.push_back((uint8_t)exact);
                out->cons.push_back(c);
                out->prod.push_back(p);
                out->dly.push_back(d);
            } else if (key.is("synapse")) {
                if (args.size() != 2) return ferr("'synapse' needs 2 fields");
                long long a = 0, b = 0;
                if (int rc = get_index(0, count, &a)) return rc;
                if (int rc = get_index(1, count, &b)) return rc;
                if (a == b) return efail(SNPIO_ERR_REFLEXIVE, "synapse (%lld, %lld) is reflexive", a, a);
                out->syn.push_back(((unsigned long long)a << 32) | (unsigned long long)b);
            } else {
                if (int rc = get_index(0, count, &out->output)) return rc;
            }
        } else {
            return ferr("unknown directive %s", key.repr().c_str());
        }
        return SNPIO_OK;
    }

    // Lines of text[i, len) until the end, an error, or (stop_after_spikes)
    // the line after 'spikes'; returns the offset reached.
    size_t scan(const char* text, size_t i, size_t len, bool stop_after_spikes) {
        while (i < len) {
            size_t e = i;
            while (e < len && !is_break((unsigned char)text[e])) ++e;
            const char* raw = text + i;
            const size_t raw_n = e - i;
            size_t next = e;  // str.splitlines: \r\n counts once
            if (next < len) next += (text[next] == '\r' && next + 1 < len && text[next + 1] == '\n') ? 2 : 1;
            i = next;
            if (line(raw, raw_n) != SNPIO_OK) return i;
            if (stop_after_spikes && spikes) return i;
        }
        return i;
    }

    int run(const char* text, size_t len) {
        Sink main_sink;
        out = &main_sink;
        size_t i = scan(text, 0, len, true);
        if (err_code) return fail(err_code, "%s", err.c_str());
        // the rest (rules, synapses, output) in parallel chunks cut at '\n'
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const size_t rest = len - i;
        // SNPIO_PARSE_CHUNK_BYTES: smallest chunk (tests shrink it to exercise the split)
        size_t chunk = 1u << 20;
        if (const char* e = getenv("SNPIO_PARSE_CHUNK_BYTES")) chunk = std::max<size_t>(1, strtoull(e, nullptr, 10));
        const size_t nt = rest < 4 * chunk ? 1 : std::min<size_t>(hw, rest / chunk);
        std::vector<size_t> cut(nt + 1, len);
        cut[0] = i;
        for (size_t c = 1; c < nt; ++c) {
            size_t x = std::max(cut[c - 1], i + rest * c / nt);
            while (x < len && text[x] != '\n') ++x;
            cut[c] = x < len ? x + 1 : len;
        }
        // chunks count their own lines; the first failing one is re-parsed
        // below with its absolute line number
        std::vector<Parser> ps(nt);
        std::vector<Sink> sinks(nt);
        for (size_t c = 0; c < nt; ++c) {
            ps[c].m = m;
            ps[c].out = &sinks[c];
            ps[c].header = header;
            ps[c].spikes = spikes;
            ps[c].count = count;
            const size_t bytes = cut[c + 1] - cut[c];
            sinks[c].syn.reserve(bytes / 16);  // growth copies cost more than untouched reserve
        }
        for_each_index(nt, nt, [&](size_t c, size_t) { ps[c].scan(text, cut[c], cut[c + 1], false); });
        long long base = lineno;
        for (size_t c = 0; c < nt; ++c) {
            if (ps[c].err_code) {
                Sink scratch;
                Parser r;
                r.m = m;
                r.out = &scratch;
                r.header = header;
                r.spikes = spikes;
                r.count = count;
                r.lineno = base;
                r.scan(text, cut[c], cut[c + 1], false);
                return fail(r.err_code, "%s", r.err.c_str());
            }
            base += ps[c].lineno;
        }
        if (!header) return fail(SNPIO_ERR_FORMAT, "empty model file");
        if (count < 0 || !spikes) return fail(SNPIO_ERR_FORMAT, "model file is missing 'neurons' or 'spikes'");
        // rules in file order: one thread per field
        m->initial.swap(main_sink.initial);
        m->output = main_sink.output;
        for (const Sink& k : sinks)
            if (k.output >= 0) m->output = k.output;
        auto concat = [&](auto field, auto& dstv) {
            size_t n = 0;
            for (Sink& k : sinks) n += (k.*field).size();
            dstv.resize(n);
            size_t at = 0;
            for (Sink& k : sinks) {
                auto& v = k.*field;
                std::copy(v.begin(), v.end(), dstv.begin() + at);
                at += v.size();
                std::remove_reference_t<decltype(v)>().swap(v);
            }
        };
        for_each_index(6, 6, [&](size_t f, size_t) {
            switch (f) {
                case 0: concat(&Sink::owner, m->owner); break;
                case 1: concat(&Sink::thr, m->thr); break;
                case 2: concat(&Sink::cons, m->cons); break;
                case 3: concat(&Sink::prod, m->prod); break;
                case 4: concat(&Sink::dly, m->dly); break;
                default: concat(&Sink::exact, m->exact); break;
            }
        });
        return finish((size_t)count, sinks);
    }

    // validate(): synapses -> ascending, de-duplicated CSR
    int finish(size_t q, std::vector<Sink>& sinks) {
        std::vector<long long>& off = m->adj_off;
        off.assign(q + 1, 0);
        size_t total = 0;
        for (const Sink& k : sinks) {
            total += k.syn.size();
            for (unsigned long long x : k.syn) off[(x >> 32) + 1]++;
        }
        for (size_t v = 0; v < q; ++v) off[v + 1] += off[v];
        std::vector<uint32_t> dst(total);
        {
            std::vector<long long> cur(off.begin(), off.end() - 1);
            for (Sink& k : sinks) {
                for (unsigned long long x : k.syn) dst[(size_t)cur[x >> 32]++] = (uint32_t)x;
                std::vector<unsigned long long>().swap(k.syn);
            }
        }
        // per-neuron sort + unique, then compaction, over neuron ranges
        const size_t nt = total < (1u << 20) ? 1 : std::max(1u, std::thread::hardware_concurrency());
        std::vector<long long> kept(q + 1, 0);
        for_each_index(q, nt, [&](size_t v, size_t) {
            auto b = dst.begin() + off[v], e = dst.begin() + off[v + 1];
            std::sort(b, e);
            kept[v + 1] = (long long)(std::unique(b, e) - b);
        });
        for (size_t v = 0; v < q; ++v) kept[v + 1] += kept[v];
        m->adj_dst.resize((size_t)kept[q]);
        for_each_index(q, nt, [&](size_t v, size_t) {
            std::copy(dst.begin() + off[v], dst.begin() + off[v] + (kept[v + 1] - kept[v]),
                      m->adj_dst.begin() + kept[v]);
        });
        off.swap(kept);
        return SNPIO_OK;
    }
};

// ---- writer

struct Out {
    FILE* f;
    std::vector<char> buf;
    size_t n = 0;
    explicit Out(FILE* f_) : f(f_), buf(1 << 22) {}
    bool flush() {
        if (n && fwrite(buf.data(), 1, n, f) != n) return false;
        n = 0;
        return true;
    }
    bool room(size_t k) { return (buf.size() - n >= k) || flush(); }
    void put(const char* s) {
        while (*s) buf[n++] = *s++;
    }
    void put(char c) { buf[n++] = c; }
    void num(long long v) {
        char t[24];
        int k = 0;
        unsigned long long u = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
        do {
            t[k++] = (char)('0' + u % 10);
            u /= 10;
        } while (u);
        if (v < 0) buf[n++] = '-';
        while (k) buf[n++] = t[--k];
    }
};

}  // namespace

extern "C" {

const char* snpio_last_error(void) { return g_err.c_str(); }

int snpio_parse(const char* text, int64_t len, snpio_model** out) {
    if (!out || (!text && len > 0) || len < 0) return fail(SNPIO_ERR_IO, "bad arguments");
    *out = nullptr;
    try {
        auto* m = new snpio_model();
        Parser p;
        p.m = m;
        int rc = p.run(text, (size_t)len);
        if (rc != SNPIO_OK) {
            delete m;
            return rc;
        }
        *out = m;
        return SNPIO_OK;
    } catch (const std::bad_alloc&) {
        return fail(SNPIO_ERR_NOMEM, "out of host memory while parsing the model file");
    }
}

int snpio_parse_file(const char* path, snpio_model** out) {
    if (!path || !out) return fail(SNPIO_ERR_IO, "bad arguments");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(SNPIO_ERR_IO, "cannot open %s: %s", path, strerror(errno));
    std::vector<char> data;
    try {
        if (fseek(f, 0, SEEK_END) == 0) {
            const long sz = ftell(f);
            if (sz > 0) data.resize((size_t)sz);
            fseek(f, 0, SEEK_SET);
        }
        size_t got = data.empty() ? 0 : fread(data.data(), 1, data.size(), f);
        data.resize(got);
    } catch (const std::bad_alloc&) {
        fclose(f);
        return fail(SNPIO_ERR_NOMEM, "out of host memory reading %s", path);
    }
    fclose(f);
    return snpio_parse(data.data(), (int64_t)data.size(), out);
}

int snpio_model_sizes(const snpio_model* m, int64_t* q, int64_t* nr, int64_t* s, int64_t* output) {
    if (!m) return fail(SNPIO_ERR_IO, "null model");
    if (q) *q = (int64_t)m->initial.size();
    if (nr) *nr = (int64_t)m->owner.size();
    if (s) *s = (int64_t)m->adj_dst.size();
    if (output) *output = m->output;
    return SNPIO_OK;
}

int snpio_model_export(const snpio_model* m, int64_t* initial, int64_t* offsets, int64_t* threshold,
                       uint8_t* is_exact, int64_t* consumed, int64_t* produced, int64_t* delay,
                       int64_t* adj_offsets, int64_t* adj_targets) {
    if (!m) return fail(SNPIO_ERR_IO, "null model");
    const size_t q = m->initial.size(), nr = m->owner.size();
    if (initial) std::copy(m->initial.begin(), m->initial.end(), initial);
    // stable regroup of rules by owner (validate(), model.py:251)
    std::vector<long long> off(q + 1, 0);
    for (uint32_t o : m->owner) off[o + 1]++;
    for (size_t v = 0; v < q; ++v) off[v + 1] += off[v];
    if (offsets) std::copy(off.begin(), off.end(), offsets);
    std::vector<long long> cur(off.begin(), off.end() - (q ? 1 : 0));
    for (size_t r = 0; r < nr; ++r) {
        const size_t at = (size_t)cur[m->owner[r]]++;
        if (threshold) threshold[at] = m->thr[r];
        if (is_exact) is_exact[at] = m->exact[r];
        if (consumed) consumed[at] = m->cons[r];
        if (produced) produced[at] = m->prod[r];
        if (delay) delay[at] = m->dly[r];
    }
    if (adj_offsets) std::copy(m->adj_off.begin(), m->adj_off.end(), adj_offsets);
    if (adj_targets) std::copy(m->adj_dst.begin(), m->adj_dst.end(), adj_targets);
    return SNPIO_OK;
}

void snpio_model_free(snpio_model* m) { delete m; }

int snpio_write_file(const char* path, int64_t q, int64_t m, int64_t s, const int64_t* initial,
                     const int64_t* offsets, const int64_t* threshold, const uint8_t* is_exact,
                     const int64_t* consumed, const int64_t* produced, const int64_t* delay,
                     const int64_t* adj_offsets, const int64_t* adj_targets, int64_t output) {
    if (!path || q < 0 || m < 0 || s < 0) return fail(SNPIO_ERR_IO, "bad arguments");
    if ((q && (!initial || !offsets || !adj_offsets)) || (m && (!threshold || !is_exact || !consumed || !produced || !delay)) ||
        (s && !adj_targets))
        return fail(SNPIO_ERR_IO, "missing arrays");
    FILE* f = fopen(path, "wb");
    if (!f) return fail(SNPIO_ERR_IO, "cannot open %s: %s", path, strerror(errno));
    bool ok = true;
    try {
        Out o(f);
        ok = o.room(64);
        o.put("snp 1\nneurons ");
        o.num(q);
        o.put("\nspikes");
        for (int64_t i = 0; ok && i < q; ++i) {
            ok = o.room(32);
            o.put(' ');
            o.num(initial[i]);
        }
        o.put('\n');
        for (int64_t v = 0; ok && v < q; ++v) {
            for (int64_t r = offsets[v]; ok && r < offsets[v + 1]; ++r) {
                ok = o.room(160);
                o.put("rule ");
                o.num(v + 1);
                o.put(is_exact[r] ? " eq " : " ge ");
                o.num(threshold[r]);
                o.put(' ');
                o.num(consumed[r]);
                o.put(' ');
                o.num(produced[r]);
                o.put(' ');
                o.num(delay[r]);
                o.put('\n');
            }
        }
        for (int64_t v = 0; ok && v < q; ++v) {
            for (int64_t x = adj_offsets[v]; ok && x < adj_offsets[v + 1]; ++x) {
                ok = o.room(64);
                o.put("synapse ");
                o.num(v + 1);
                o.put(' ');
                o.num(adj_targets[x] + 1);
                o.put('\n');
            }
        }
        if (ok && output >= 0) {
            ok = o.room(32);
            o.put("output ");
            o.num(output + 1);
            o.put('\n');
        }
        ok = ok && o.flush();
    } catch (const std::bad_alloc&) {
        fclose(f);
        return fail(SNPIO_ERR_NOMEM, "out of host memory writing %s", path);
    }
    if (fclose(f) != 0) ok = false;
    return ok ? SNPIO_OK : fail(SNPIO_ERR_IO, "write to %s failed", path);
}

int snpio_write_trace(const char* path, const int64_t* rows, int64_t n_rows, int64_t q, int32_t append) {
    if (!path || n_rows < 0 || q < 0 || (n_rows && q && !rows)) return fail(SNPIO_ERR_IO, "bad arguments");
    FILE* f = fopen(path, append ? "ab" : "wb");
    if (!f) return fail(SNPIO_ERR_IO, "cannot open %s: %s", path, strerror(errno));
    bool ok = true;
    try {
        Out o(f);
        for (int64_t r = 0; ok && r < n_rows; ++r) {
            const int64_t* row = rows + r * q;
            for (int64_t i = 0; ok && i < q; ++i) {
                ok = o.room(24);
                if (i) o.put(' ');
                o.num(row[i]);
            }
            ok = ok && o.room(2);
            o.put('\n');
        }
        ok = ok && o.flush();
    } catch (const std::bad_alloc&) {
        fclose(f);
        return fail(SNPIO_ERR_NOMEM, "out of host memory writing %s", path);
    }
    if (fclose(f) != 0) ok = false;
    return ok ? SNPIO_OK : fail(SNPIO_ERR_IO, "write to %s failed", path);
}

}  // extern "C"

// ---- synthetic family synth-v1 (generators.py synth_v1, synth_v1_rows)

namespace {

inline uint64_t mix64_h(uint64_t seed, int64_t stream, int64_t i) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(stream + 1) + 0xBF58476D1CE4E5B9ull * (uint64_t)(i + 1);
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

constexpr int kSynthDegree = 16;

// the 16 ascending out-neighbours of source i
inline void synth_targets(int64_t q, uint64_t seed, int64_t i, int64_t* t) {
    const int64_t w = (q - 1) / kSynthDegree;
    for (int k = 0; k < kSynthDegree; ++k)
        t[k] = (i + 1 + k * w + (int64_t)(mix64_h(seed, 1 + k, i) % (uint64_t)w)) % q;
    std::sort(t, t + kSynthDegree);
}

template <typename F>
void parallel_for(int64_t n, F f) {
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>((int64_t)std::thread::hardware_concurrency(), n / 65536 + 1));
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back([=] {
            const int64_t a = n * t / nt, b = n * (t + 1) / nt;
            f(a, b);
        });
    for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int snpio_synth_v1_edges(int64_t q, uint64_t seed, int64_t lo, int64_t hi, int64_t* n_edges) {
    if (q < kSynthDegree + 1 || lo < 0 || hi > q || lo > hi || !n_edges) return fail(SNPIO_ERR_IO, "bad arguments");
    if (lo == 0 && hi == q) {
        *n_edges = kSynthDegree * q;
        return SNPIO_OK;
    }
    std::vector<int64_t> part(std::max<unsigned>(1, std::thread::hardware_concurrency()) + 1, 0);
    const int64_t nt = (int64_t)part.size() - 1;
    std::vector<std::thread> th;
    for (int64_t t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            int64_t c = 0, tg[kSynthDegree];
            for (int64_t i = q * t / nt; i < q * (t + 1) / nt; ++i) {
                synth_targets(q, seed, i, tg);
                for (int k = 0; k < kSynthDegree; ++k) c += tg[k] >= lo && tg[k] < hi;
            }
            part[t] = c;
        });
    for (auto& x : th) x.join();
    int64_t tot = 0;
    for (int64_t t = 0; t < nt; ++t) tot += part[t];
    *n_edges = tot;
    return SNPIO_OK;
}

int snpio_synth_v1(int64_t q, uint64_t seed, int32_t delays, int64_t lo, int64_t hi, int64_t* initial,
                   int64_t* offsets, int64_t* threshold, uint8_t* is_exact, int64_t* consumed, int64_t* produced,
                   int64_t* delay, int64_t* adj_offsets, int64_t* adj_targets) {
    if (q < kSynthDegree + 1 || lo < 0 || hi > q || lo > hi) return fail(SNPIO_ERR_IO, "bad arguments");
    const int64_t n = hi - lo;
    // rows [lo, hi): initial spikes and the four rules (generators.py synth_v1)
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r) {
            const int64_t i = lo + r;
            initial[r] = (int64_t)(mix64_h(seed, 0, i) % 8);
            const int64_t t0 = 2 + (int64_t)(mix64_h(seed, 17, i) % 4), t1 = 3 + (int64_t)(mix64_h(seed, 18, i) % 6);
            const int64_t c1 = 1 + (int64_t)(mix64_h(seed, 19, i) % (uint64_t)t1), t2 = 1 + (int64_t)(mix64_h(seed, 20, i) % 5);
            const int64_t thr[4] = {t0, t1, t2, 1}, con[4] = {t0, c1, t2, 1}, pro[4] = {1, 1, 0, 1};
            const uint8_t ex[4] = {1, 0, 1, 0};
            int64_t dl[4] = {0, 0, 0, 0};
            if (delays) {
                dl[0] = (int64_t)(mix64_h(seed, 21, i) % 4);
                dl[1] = (int64_t)(mix64_h(seed, 22, i) % 4);
                dl[3] = (int64_t)(mix64_h(seed, 23, i) % 4);
            }
            for (int k = 0; k < 4; ++k) {
                threshold[4 * r + k] = thr[k];
                is_exact[4 * r + k] = ex[k];
                consumed[4 * r + k] = con[k];
                produced[4 * r + k] = pro[k];
                delay[4 * r + k] = dl[k];
            }
            offsets[r] = 4 * r;
        }
    });
    offsets[n] = 4 * n;
    // adjacency over all q sources, edges entering [lo, hi), ascending targets
    if (lo == 0 && hi == q) {
        parallel_for(q, [&](int64_t a, int64_t b) {
            for (int64_t i = a; i < b; ++i) {
                synth_targets(q, seed, i, adj_targets + kSynthDegree * i);
                adj_offsets[i] = kSynthDegree * i;
            }
        });
        adj_offsets[q] = kSynthDegree * q;
        return SNPIO_OK;
    }
    std::vector<int64_t> cnt(q + 1, 0);
    parallel_for(q, [&](int64_t a, int64_t b) {
        int64_t tg[kSynthDegree];
        for (int64_t i = a; i < b; ++i) {
            synth_targets(q, seed, i, tg);
            int64_t c = 0;
            for (int k = 0; k < kSynthDegree; ++k) c += tg[k] >= lo && tg[k] < hi;
            cnt[i] = c;
        }
    });
    adj_offsets[0] = 0;
    for (int64_t i = 0; i < q; ++i) adj_offsets[i + 1] = adj_offsets[i] + cnt[i];
    parallel_for(q, [&](int64_t a, int64_t b) {
        int64_t tg[kSynthDegree];
        for (int64_t i = a; i < b; ++i) {
            if (!cnt[i]) continue;
            synth_targets(q, seed, i, tg);
            int64_t w = adj_offsets[i];
            for (int k = 0; k < kSynthDegree; ++k)
                if (tg[k] >= lo && tg[k] < hi) adj_targets[w++] = tg[k];
        }
    });
    return SNPIO_OK;
}

}  // extern "C"
