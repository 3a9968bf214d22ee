/*
 * snpb200.h -- C ABI of the B200 SNP-system step engine (libsnpb200.so).
 *
 * The reference (snpsim 0.1.0, pure Python + numpy) has no FFI; its plug
 * point is the hard-coded format dispatch inside the engine:
 *
 *   prepare()            pkg/src/snpsim/engine.py:388-402   -> snp_engine_create
 *   simulate_prepared()  pkg/src/snpsim/engine.py:416-461   -> snp_begin + snp_advance
 *                                                               (snp_run = both + final read)
 *   sv_calc()            pkg/src/snpsim/engine.py:192-236   -> snp_sv_calc
 *   step_sparse/_ell/_compressed()
 *                        pkg/src/snpsim/engine.py:239-355   -> snp_step
 *   update_delays()      pkg/src/snpsim/engine.py:358-366   -> snp_update_delays
 *   NegativeSpikes       pkg/src/snpsim/engine.py:48-54     -> SNP_ERR_NEGATIVE
 *
 * Every entry point takes plain HOST pointers in the reference's own array
 * layouts (int64 counts, numpy-bool kinds, NULL = -1 padding) and sizes; the
 * library owns all device memory.  No torch / CUDA types cross the boundary
 * (streams are internal; one stream per engine).  An engine is not
 * re-entrant (same contract as the reference engine).
 *
 * Return codes: 0 ok; SNP_ERR_NEGATIVE -> NegativeSpikes; SNP_ERR_BAD_ARG ->
 * ValueError; SNP_ERR_CUDA / SNP_ERR_CAPACITY -> RuntimeError / MemoryError.
 * snp_last_error() returns the thread's last message.
 */
#ifndef SNPB200_H
#define SNPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNPB200_ABI_VERSION 6

enum {
    SNP_OK = 0,
    SNP_ERR_NEGATIVE = 1,
    SNP_ERR_BAD_ARG = 2,
    SNP_ERR_CUDA = 3,
    SNP_ERR_CAPACITY = 4
};

/* matrices.py:33-45 Format (ORACLE has no device backend) */
enum { SNP_FMT_SPARSE = 0, SNP_FMT_ELL = 1, SNP_FMT_COMPRESSED = 2 };

/* COMPRESSED only: TILED (default) = destination tiles with source-sorted
 * in-edge segments and shared-memory accumulation; PULL = per-destination
 * CSR gather; PUSH = the paper's Alg. 5 scatter with atomics. */
enum { SNP_VARIANT_AUTO = 0, SNP_VARIANT_PULL = 1, SNP_VARIANT_PUSH = 2, SNP_VARIANT_TILED = 3,
       SNP_VARIANT_TILED2 = 4,    /* TILED2: two-pass receive (pass 1 per source window, then tiles);
                                     for sources spread far beyond the engine's rows (10^8, partitions) */
       SNP_VARIANT_SMALL = 5 };   /* SMALL: q <= 16384 -- one CTA runs a whole loop segment per launch
                                     (no per-step launch); AUTO picks it for small systems */

/* selection.py:21-31 */
enum { SNP_POLICY_FIRST = 0, SNP_POLICY_SEEDED = 1 };

/* engine.py:57-60 RecordLevel as bit flags; 0 = final state only
 * (extension used by the benchmark). CONFIGS=1, CONFIGS_AND_DELAYS=3, FULL=7. */
enum { SNP_REC_CONFIGS = 1, SNP_REC_DELAYS = 2, SNP_REC_SPIKING = 4 };
/* Extension: with SNP_REC_DIGEST the recorded rows stay on the device and
 * snp_advance returns one 64-bit digest per row instead (large recorded
 * runs: 8 bytes per row instead of 8q).  digest(row) = sum over j of
 * fmix64(v_j * 0x9E3779B97F4A7C15 + (j + 1) * 0xD6E8FEB86659FD93) mod 2^64,
 * fmix64 the SplitMix64 finaliser of selection.py:37-45, v_j the int64 value
 * (config count, delay, chosen rule id or -1). */
enum { SNP_REC_DIGEST = 8 };

/* engine.py:57-59 HaltReason */
enum { SNP_RUNNING = 0, SNP_HALT_STEP_LIMIT = 1, SNP_HALT_NO_APPLICABLE = 2,
       SNP_HALT_NEGATIVE = 3, SNP_HALT_EXCHANGE = 4 };

typedef struct snp_system_desc {
    int32_t format;            /* SNP_FMT_* */
    int32_t variant;           /* SNP_VARIANT_* */
    int64_t q;                 /* neurons */
    int64_t m;                 /* rules */
    const int64_t *initial;    /* [q]   SNPSystem.initial_spikes           */
    const int64_t *offsets;    /* [q+1] NeuronRuleMap.offsets              */
    const int64_t *threshold;  /* [m]   RuleVector.threshold               */
    const uint8_t *is_exact;   /* [m]   RuleVector.is_exact (numpy bool)   */
    const int64_t *consumed;   /* [m]   RuleVector.consumed                */
    const int64_t *produced;   /* [m]   RuleVector.produced                */
    const int64_t *delay;      /* [m]   RuleVector.delay                   */
    /* Transition structure.  Either the out-adjacency in CSR form
     * (ascending targets per source), or -- when adj_offsets is NULL -- the
     * reference matrix of the chosen format in its own layout:           */
    const int64_t *adj_offsets;  /* [q+1] */
    const int64_t *adj_targets;  /* [S]   */
    const int64_t *syn_target;   /* SynapseMatrix.target [syn_rows][q] (matrices.py:100-112) */
    int64_t syn_rows;
    const int64_t *ell_target;   /* EllMatrix.target [ell_rows][m] (matrices.py:83-97) */
    const int64_t *ell_amount;   /* EllMatrix.amount [ell_rows][m] */
    int64_t ell_rows;
    const int64_t *sparse_data;  /* SparseMatrix.data [m][q] (matrices.py:76-80) */
    int32_t device;              /* CUDA ordinal */
    int32_t world;               /* row partition: ranks (0 or 1 = whole system) */
    int32_t rank;                /* row partition: this engine's rank */
    int32_t x_pbits;             /* row partition: P element width agreed by every rank:
                                    1 (bits; every sending rule produces x_pmax), 8, 16 or 32;
                                    0 = decided from this rank's own rules */
    int64_t x_pmax;              /* row partition: largest produced amount over all ranks */
} snp_system_desc;

typedef struct snp_run_opts {
    int64_t max_steps;     /* SimOptions.max_steps (>= 1) */
    int32_t policy;        /* SNP_POLICY_* */
    int32_t record;        /* SNP_REC_* flags */
    uint64_t seed;         /* SeededRandom.seed mod 2^64 */
    int64_t chunk;         /* steps per device loop segment (0 = auto) */
    int32_t use_graph;     /* 1 = replay segments from a CUDA graph */
    int32_t collect_stats; /* 1 = accumulate traffic counters (snp_result.stats) */
} snp_run_opts;

/* Host output rows for snp_advance.  Row i holds step (first_row_step + i):
 * configs/delays are C_k/D_k (configs[k] of engine.py:143), spiking the
 * chosen-rule ids of step k (-1 = none).  Any pointer may be NULL. */
typedef struct snp_trace_out {
    int64_t *configs;  /* [cap][q] */
    int64_t *delays;   /* [cap][q] */
    int64_t *spiking;  /* [cap][q] */
    int64_t cap;       /* rows available */
    int64_t first_row_step;  /* out: step of row 0 */
    int64_t config_rows;     /* out: rows of configs/delays written */
    int64_t spiking_rows;    /* out: rows of spiking written */
    uint64_t *config_digests;  /* [cap] with SNP_REC_DIGEST (may be NULL) */
    uint64_t *delay_digests;   /* [cap] */
    uint64_t *spiking_digests; /* [cap] */
} snp_trace_out;

enum {
    SNP_STAT_STEPS = 0,     /* steps executed with selection */
    SNP_STAT_SCANNED,       /* sum over open neurons of rules scanned */
    SNP_STAT_FIRED,         /* |F| */
    SNP_STAT_SENDING,       /* fired with p > 0 */
    SNP_STAT_EDGES,         /* adjacency entries read (gathered or pushed) */
    SNP_STAT_ROWS,          /* reference walk rows: sum over sending of e + [e < z] */
    SNP_STAT_OPEN,          /* open neurons (sum over steps) */
    SNP_STAT_COUNT
};

typedef struct snp_result {
    int64_t steps;         /* Trace.steps */
    int32_t halt;          /* SNP_RUNNING / SNP_HALT_* */
    int32_t error;         /* SNP_OK or SNP_ERR_NEGATIVE */
    int64_t negative_neuron;  /* first neuron seen negative (error only) */
    int64_t negative_value;
    uint64_t stats[SNP_STAT_COUNT];
    int64_t kernel_launches;  /* device kernels launched by this call */
} snp_result;

typedef struct snp_engine snp_engine;

typedef struct snp_engine_info {
    int64_t q, m, z;
    int64_t device_bytes;     /* device memory held by the engine */
    int32_t format, variant;
    int32_t p_mode;           /* 0 bit (p common), 1 u8, 2 u16, 3 u32 */
    int32_t heavy_neurons;
    int64_t in_edges;         /* pull: padded in-adjacency entries; tiled: segment words */
    int64_t p_common;
    int64_t tile;             /* tiled: destinations per tile */
    int64_t n_tiles;
    int32_t ring_stages;      /* tiled: TMA ring stages in shared memory */
    int32_t counter_bits;     /* tiled: 16 or 32-bit destination counters */
    int64_t stage_bytes;      /* tiled: bytes per ring stage */
    int32_t push_kernel;      /* ELL / COMPRESSED-push runs: SNP_PUSH_* */
    int32_t push_tiles;       /* SNP_PUSH_BINNED: destination tiles (bins) */
} snp_engine_info;

/* snp_engine_info.push_kernel: how a push-format run steps */
enum { SNP_PUSH_NONE = 0,      /* pull formats / dense */
       SNP_PUSH_UNFUSED = 1,   /* step kernel + scatter kernels (heavy-rule neurons, SNPB200_PUSH=unfused) */
       SNP_PUSH_ATOMIC = 2,    /* one kernel, L2 RED.ADD into a receive array */
       SNP_PUSH_BINNED = 3 };  /* one kernel, deliveries binned by destination tile (ell_bin_step_kernel) */

int snp_abi_version(void);
const char *snp_last_error(void);
int snp_device_count(void);

int snp_engine_create(const snp_system_desc *desc, snp_engine **out);
void snp_engine_destroy(snp_engine *eng);
int snp_engine_get_info(const snp_engine *eng, snp_engine_info *info);

/* Reset the run state to `initial` (int64 [q] in host memory or, through
 * unified addressing, in device memory -- e.g. a torch CUDA tensor; NULL =
 * the system's own initial configuration) with every neuron open
 * (engine.py:427-428). */
int snp_begin(snp_engine *eng, const int64_t *initial);
/* Execute up to `n_steps` more steps of the loop of engine.py:441-458,
 * stopping early on halt / error or when `trace` (may be NULL) is full. */
int snp_advance(snp_engine *eng, const snp_run_opts *opts, int64_t n_steps,
                snp_trace_out *trace, snp_result *res);
/* Final state after a halt: C and D (int64 [q] each, host or device memory;
 * either may be NULL). */
int snp_read_state(snp_engine *eng, int64_t *config, int64_t *delays);
/* snp_begin + snp_advance(to halt) + snp_read_state. */
int snp_run(snp_engine *eng, const int64_t *initial, const snp_run_opts *opts,
            int64_t *final_config, int64_t *final_delays, snp_result *res);
/* Device-resident time of the last snp_advance/snp_run device loop (ms). */
double snp_last_device_ms(const snp_engine *eng);

/* Phase functions (engine.py:192-366), host arrays in, host arrays out. */
int snp_sv_calc(snp_engine *eng, const int64_t *config, const int64_t *delays,
                int32_t policy, uint64_t seed, int64_t step, int64_t *chosen);
int snp_step(snp_engine *eng, const int64_t *config, const int64_t *delays,
             const int64_t *chosen, int64_t *next_config, int64_t *row_visits);
int snp_update_delays(snp_engine *eng, const int64_t *delays, const int64_t *chosen,
                      int64_t *next_delays);

/* Row partition (multi-GPU).  An engine created with
 * world > 1 owns neurons [lo, hi) of the q-neuron system, COMPRESSED only,
 * with nl = round_up(ceil(q / world), 128), lo = rank * nl, hi = min(q, lo + nl).
 * In the descriptor, `q` is the whole system, the node arrays (initial,
 * offsets, rule vector, `m`) describe neurons [lo, hi) only, and
 * adj_offsets/adj_targets is a CSR over all q sources that must contain every
 * edge entering [lo, hi) (other edges are ignored).  Each step kernel
 * publishes the rank's production bits and step flags into its chunk of the
 * current exchange slot; the caller must all-gather that slot across ranks
 * (in place: chunk at chunk_offset_bytes of a slot_bytes buffer) before the
 * next snp_launch_step.  Step k writes slot k % 3. */
typedef struct snp_exchange {
    void *slot[3];               /* device pointers of the three exchange slots */
    int64_t slot_bytes;          /* bytes all-gathered per slot */
    int64_t chunk_offset_bytes;  /* this rank's chunk within a slot */
    int64_t chunk_bytes;
    int64_t lo, hi;              /* owned global neurons */
    int64_t neurons_per_rank;
    int32_t world, rank;
} snp_exchange;

int snp_exchange_info(const snp_engine *eng, snp_exchange *x);
/* Launch on the caller's CUDA stream (cudaStream_t passed as void*; NULL =
 * the engine's own stream), e.g. the stream NCCL runs on. */
int snp_set_stream(snp_engine *eng, void *stream);
/* After snp_begin: run parameters for snp_launch_step.  With record flags
 * (SNP_REC_CONFIGS / DELAYS / SPIKING) every row of the run is kept on the
 * device (max_steps + 2 rows) for snp_read_trace. */
int snp_configure(snp_engine *eng, const snp_run_opts *opts);
/* Rows [first_row, first_row + n_rows) of a configured recording run
 * (row k = the state after k steps; this engine's neurons; chosen = this
 * engine's rule indices or -1).  Host int64 [n_rows][q] each; NULL skips. */
int snp_read_trace(snp_engine *eng, int64_t first_row, int64_t n_rows, int64_t *configs,
                   int64_t *delays, int64_t *chosen);
/* Enqueue one step (no host synchronisation). */
int snp_launch_step(snp_engine *eng);
/* Synchronise the engine stream and read the run state. */
int snp_poll(snp_engine *eng, snp_result *res);

/* Peer exchange (NVLink / NVSwitch P2P; replaces the all-gather).  Every
 * rank's step kernel stores its P chunk and step header straight into each
 * peer's exchange slot (tile by tile, overlapping the step's own work) and
 * then raises a per-rank step flag on every peer; the next step kernel waits
 * for all flags of the previous step.  No collective call per step: after
 * connecting, the caller only calls snp_launch_step.  Every rank must finish
 * snp_begin before any rank launches the run's first step (a host barrier).
 * A rank that stops stepping makes the others halt with SNP_ERR_CUDA
 * ("peer exchange timed out") after 20 s instead of hanging.
 *   snp_exchange_ipc_handle: this rank's exchange block as a CUDA IPC handle
 *     (SNP_IPC_HANDLE_BYTES bytes) to all-gather across processes;
 *   snp_exchange_connect: map every rank's block (handles[world]) into this
 *     process and enable peer exchange;
 *   snp_exchange_connect_local: the same for `world` engines of one process
 *     (e.g. several ranks on one device). */
#define SNP_IPC_HANDLE_BYTES 64
int snp_exchange_ipc_handle(const snp_engine *eng, void *handle);
int snp_exchange_connect(snp_engine *eng, const void *handles, int world);
int snp_exchange_connect_local(snp_engine *const *engines, int world);

/* Diagnostics: digests of the tiled layout arrays (segment words, segment
 * bases, stage descriptors, tile->stage and tile->segment ranges, stage
 * bases), row_digest-style sums; equal digests = identical layouts (the
 * device build and the host reference build are checked this way). */
int snp_engine_layout_digest(const snp_engine *eng, uint64_t *out /* [6] */);

/* Timing helper for benchmarks: run `steps` steps (no recording) from the
 * current state with the device loop only and return the per-kernel mean
 * duration of the dominant step kernel in *kernel_ms (CUDA events around
 * each launch on the engine stream) and the total in *total_ms. */
int snp_time_steps(snp_engine *eng, const snp_run_opts *opts, int64_t steps,
                   double *total_ms, double *kernel_ms, snp_result *res);

#ifdef __cplusplus
}
#endif

#endif /* SNPB200_H */
