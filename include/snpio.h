/*
 * snpio.h -- native model-file I/O (libsnpio.so, host only).
 *
 * Replaces the reference's line-by-line text parser and writer,
 * pkg/src/snpsim/modelfile.py:40-57 (serialize_model) and :60-143
 * (parse_model), for systems too large to hold as one Python object per
 * rule and synapse.  The parser applies the reference's checks in the
 * reference's order and reports them with the same messages; the result is
 * the validated system as flat arrays in the C ABI layout of snpb200.h
 * (rules grouped by owner in file order, synapses ascending and de-duplicated).
 *
 * Return codes map to the reference's exception types:
 *   0 ok, 1 ModelFileError, 2 InvalidRule, 3 UnknownNeuron,
 *   4 ReflexiveSynapse, 5 ModelError, 6 I/O error, 7 out of memory.
 * snpio_last_error() returns the thread's last message.
 */
#ifndef SNPIO_H
#define SNPIO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SNPIO_OK = 0,
    SNPIO_ERR_FORMAT = 1,
    SNPIO_ERR_INVALID_RULE = 2,
    SNPIO_ERR_UNKNOWN_NEURON = 3,
    SNPIO_ERR_REFLEXIVE = 4,
    SNPIO_ERR_MODEL = 5,
    SNPIO_ERR_IO = 6,
    SNPIO_ERR_NOMEM = 7
};

typedef struct snpio_model snpio_model;

const char *snpio_last_error(void);

/* parse_model (modelfile.py:60-143) on a text buffer / a file */
int snpio_parse(const char *text, int64_t len, snpio_model **out);
int snpio_parse_file(const char *path, snpio_model **out);

/* q neurons, m rules, s synapses, output neuron (0-based, -1 = none) */
int snpio_model_sizes(const snpio_model *mdl, int64_t *q, int64_t *m, int64_t *s, int64_t *output);

/* Copy the arrays out: initial[q], offsets[q+1], threshold[m], is_exact[m]
 * (one byte each), consumed[m], produced[m], delay[m], adj_offsets[q+1],
 * adj_targets[s]. */
int snpio_model_export(const snpio_model *mdl, int64_t *initial, int64_t *offsets, int64_t *threshold,
                       uint8_t *is_exact, int64_t *consumed, int64_t *produced, int64_t *delay,
                       int64_t *adj_offsets, int64_t *adj_targets);

void snpio_model_free(snpio_model *mdl);

/* serialize_model (modelfile.py:40-57) of a validated system in array form,
 * written to `path`. */
int snpio_write_file(const char *path, int64_t q, int64_t m, int64_t s, const int64_t *initial,
                     const int64_t *offsets, const int64_t *threshold, const uint8_t *is_exact,
                     const int64_t *consumed, const int64_t *produced, const int64_t *delay,
                     const int64_t *adj_offsets, const int64_t *adj_targets, int64_t output);

/* format_trace (engine.py:162-165): `n_rows` configuration rows of q
 * counts, one line each, space-separated; append = 1 adds to the file
 * (a trace written segment by segment is byte-identical). */
int snpio_write_trace(const char *path, const int64_t *rows, int64_t n_rows, int64_t q, int32_t append);

/* Synthetic family synth-v1 (paper_2408_04343_b200/generators.py synth_v1,
 * SURVEY.md 8(d)), generated natively with all host threads: rows [lo, hi)
 * (initial[n], offsets[n+1], 4 rules per neuron in [4n] arrays) and the CSR
 * over all q sources of the edges entering [lo, hi) (ascending targets).
 * snpio_synth_v1_edges gives the edge count to allocate. */
int snpio_synth_v1_edges(int64_t q, uint64_t seed, int64_t lo, int64_t hi, int64_t *n_edges);
int snpio_synth_v1(int64_t q, uint64_t seed, int32_t delays, int64_t lo, int64_t hi, int64_t *initial,
                   int64_t *offsets, int64_t *threshold, uint8_t *is_exact, int64_t *consumed,
                   int64_t *produced, int64_t *delay, int64_t *adj_offsets, int64_t *adj_targets);

#ifdef __cplusplus
}
#endif

#endif /* SNPIO_H */
