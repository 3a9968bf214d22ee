/*
 * snp_oracle.c -- CPU ORACLE, test infrastructure only (never the product).
 *
 * Plain-C restatement of the reference interpreter
 * (/root/reference/pkg/src/snpsim/oracle.py:21-101, selection.py:37-71) so
 * that full-size systems (10^7 neurons) can be checked bit-exactly against
 * the B200 engine in seconds.  Sequential, int64 counts, same loop and
 * halting contract as engine.py:441-458.  Built by oracle/Makefile into
 * oracle/liboracle.so; called only from tests/ and bench.py's CPU arm.
 * Pinned against the reference's own outputs by tests/test_oracle_golden.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* selection.py:37-45 */
static uint64_t mix64(uint64_t seed, int64_t step, int64_t neuron) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(step + 1) +
                 0xBF58476D1CE4E5B9ull * (uint64_t)(neuron + 1);
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

uint64_t oracle_mix64(uint64_t seed, int64_t step, int64_t neuron) { return mix64(seed, step, neuron); }

enum { OR_OK = 0, OR_NEGATIVE = 1, OR_BAD = 2 };
enum { OR_HALT_STEP_LIMIT = 1, OR_HALT_NO_APPLICABLE = 2 };

/*
 * Run from `initial` for at most max_steps steps.  Trace rows (may be NULL):
 * tr_cfg/tr_dly hold C_k/D_k for k = 0..steps (rows <= trace_cap),
 * tr_chosen the chosen rule per neuron of step k.  Rows beyond trace_cap are
 * not recorded.  Returns OR_NEGATIVE (with *neg_neuron) when a step drives a
 * count below zero (oracle.py:52-56).
 */
int oracle_run(int64_t q, const int64_t *initial, const int64_t *offsets, const int64_t *thr,
               const uint8_t *exact, const int64_t *cons, const int64_t *prod, const int64_t *dly,
               const int64_t *adj_off, const int64_t *adj_dst, int64_t max_steps, int policy,
               uint64_t seed, int64_t trace_cap, int64_t *tr_cfg, int64_t *tr_dly, int64_t *tr_chosen,
               int64_t *out_steps, int *out_halt, int64_t *final_cfg, int64_t *final_dly,
               int64_t *neg_neuron) {
    if (q < 0 || max_steps < 0) return OR_BAD;
    int64_t *cfg = malloc(sizeof(int64_t) * (q ? q : 1));
    int64_t *nxt = malloc(sizeof(int64_t) * (q ? q : 1));
    int64_t *del = calloc(q ? q : 1, sizeof(int64_t));
    int64_t *ndl = malloc(sizeof(int64_t) * (q ? q : 1));
    int64_t *chosen = malloc(sizeof(int64_t) * (q ? q : 1));
    int rc = OR_OK;
    if (!cfg || !nxt || !del || !ndl || !chosen) {
        rc = OR_BAD;
        goto done;
    }
    memcpy(cfg, initial, sizeof(int64_t) * q);
    int64_t step = 0;
    int halt = 0;
    if (tr_cfg && trace_cap > 0) memcpy(tr_cfg, cfg, sizeof(int64_t) * q);
    if (tr_dly && trace_cap > 0) memset(tr_dly, 0, sizeof(int64_t) * q);
    for (;;) {
        if (step == max_steps) {
            halt = OR_HALT_STEP_LIMIT;
            break;
        }
        /* selection: oracle.py:33-42 */
        int64_t fired = 0;
        for (int64_t n = 0; n < q; ++n) {
            chosen[n] = -1;
            if (del[n] != 0) continue;
            const int64_t c = cfg[n];
            int64_t count = 0, first = -1;
            for (int64_t r = offsets[n]; r < offsets[n + 1]; ++r) {
                const int ok = exact[r] ? (c == thr[r]) : (c >= thr[r]);
                if (ok) {
                    if (first < 0) first = r;
                    ++count;
                }
            }
            if (!count) continue;
            int64_t pick = first;
            if (policy != 0) {
                uint64_t k = mix64(seed, step, n) % (uint64_t)count;
                for (int64_t r = offsets[n]; r < offsets[n + 1]; ++r) {
                    const int ok = exact[r] ? (c == thr[r]) : (c >= thr[r]);
                    if (ok) {
                        if (k == 0) {
                            pick = r;
                            break;
                        }
                        --k;
                    }
                }
            }
            chosen[n] = pick;
            ++fired;
        }
        int any_closed = 0;
        for (int64_t n = 0; n < q && !any_closed; ++n) any_closed = del[n] != 0;
        if (!fired && !any_closed) {
            halt = OR_HALT_NO_APPLICABLE;
            break;
        }
        /* application: oracle.py:44-56 */
        memcpy(nxt, cfg, sizeof(int64_t) * q);
        for (int64_t n = 0; n < q; ++n) {
            const int64_t r = chosen[n];
            if (r < 0) continue;
            nxt[n] -= cons[r];
            const int64_t p = prod[r];
            if (p)
                for (int64_t e = adj_off[n]; e < adj_off[n + 1]; ++e) {
                    const int64_t t = adj_dst[e];
                    if (del[t] == 0) nxt[t] += p;
                }
        }
        for (int64_t n = 0; n < q; ++n)
            if (nxt[n] < 0) {
                if (neg_neuron) *neg_neuron = n;
                rc = OR_NEGATIVE;
                goto done;
            }
        /* delays: oracle.py:58-60 */
        for (int64_t n = 0; n < q; ++n) ndl[n] = chosen[n] >= 0 ? dly[chosen[n]] : (del[n] > 0 ? del[n] - 1 : 0);
        if (tr_chosen && step < trace_cap) memcpy(tr_chosen + step * q, chosen, sizeof(int64_t) * q);
        int64_t *t = cfg;
        cfg = nxt;
        nxt = t;
        t = del;
        del = ndl;
        ndl = t;
        ++step;
        if (tr_cfg && step < trace_cap) memcpy(tr_cfg + step * q, cfg, sizeof(int64_t) * q);
        if (tr_dly && step < trace_cap) memcpy(tr_dly + step * q, del, sizeof(int64_t) * q);
    }
    if (out_steps) *out_steps = step;
    if (out_halt) *out_halt = halt;
    if (final_cfg) memcpy(final_cfg, cfg, sizeof(int64_t) * q);
    if (final_dly) memcpy(final_dly, del, sizeof(int64_t) * q);
done:
    free(cfg);
    free(nxt);
    free(del);
    free(ndl);
    free(chosen);
    return rc;
}
