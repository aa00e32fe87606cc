/*
 * graphlb_b200.h -- C-ABI of libgraphlb_b200.so, the sm_100a implementation of
 * the BFS/SSSP task-distribution hot path of `graphlb` (arXiv 1711.00231).
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, and returns
 * an int status (GLB_OK == 0).  On failure a thread-local message is available
 * from glb_last_error().  Host arrays are always the reference's int64 layout
 * (graphlb/csr.py:16-21 INDEX_DTYPE = np.int64); the library's host workers
 * narrow them to 32 bits (8 bits for small weights) on the way into pinned
 * staging buffers, so PCIe carries the narrow layout, and the library owns all
 * device memory.
 *
 * Reference interfaces each entry point replaces (paths under
 * /root/reference/pkg/src/graphlb/):
 *   glb_graph_create     CsrGraph.__post_init__/_validate       csr.py:55-85
 *                        (+ the per-run `.tolist()` of csr_locals, strategies/common.py:73-82)
 *   glb_run              run_strategy                           strategies/__init__.py:17-41
 *                        run_bs / run_ep / run_wd / run_ns / run_hp
 *                        node_based.py:19, edge_based.py:31, workload.py:162,
 *                        splitting.py:102, hierarchical.py:27
 *   glb_histogram        build_histogram + compute_mdt          degrees.py:45-76
 *   glb_degree_stats     degree_stats                           degrees.py:27-32
 *   glb_split_graph      split_graph                            strategies/splitting.py:58-99
 *   glb_csr_to_coo       csr_to_coo                             csr.py:155-170
 *   glb_inclusive_scan   inclusive_scan                         scan.py:19-65
 *   glb_find_offsets     find_offsets                           strategies/workload.py:45-72
 *   glb_validate         sequential_bfs / dijkstra + verify     oracles.py:13-82, as used by
 *                        run_benchmark(verify=True)             bench.py:186-196
 *
 * Status -> Python exception mapping used by the drop-in package:
 *   GLB_EINVAL -> ValueError, GLB_ERANGE -> IndexError, GLB_EOVERFLOW -> OverflowError,
 *   GLB_ECOO_CAPACITY -> StrategyRun(status="infeasible: memory") (never raised),
 *   GLB_ECUDA / GLB_ENODEV / GLB_ENOMEM -> RuntimeError.
 */
#ifndef GRAPHLB_B200_H
#define GRAPHLB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GLB_OK 0
#define GLB_EINVAL 1
#define GLB_ERANGE 2
#define GLB_ECOO_CAPACITY 3
#define GLB_ECUDA 4
#define GLB_ENOMEM 5
#define GLB_EOVERFLOW 6
#define GLB_ENODEV 7
#define GLB_EPARSE 8   /* malformed graph file: glb_last_error() is "<line>\t<message>", line -1 = whole file */

/* strategy ids (STRATEGY_TAGS order, strategies/__init__.py:14) */
#define GLB_BS 0
#define GLB_EP 1
#define GLB_WD 2
#define GLB_NS 3
#define GLB_HP 4
/* record tag for hierarchical.py:24 FALLBACK_TAG = "WD-fallback" */
#define GLB_TAG_WD_FALLBACK 5

/* RelaxOp kinds (strategies/common.py:23-42) */
#define GLB_BFS 0
#define GLB_SSSP 1

/* host loop driving the device iterations */
#define GLB_LOOP_HOST 0  /* one host round trip per launch (exact per-launch records) */
#define GLB_LOOP_GRAPH 1 /* device-driven: CUDA graph with a conditional WHILE node */

typedef struct glb_graph glb_graph;

typedef struct glb_run_params {
  int32_t strategy;        /* GLB_BS..GLB_HP */
  int32_t algo;            /* GLB_BFS / GLB_SSSP */
  int64_t source;          /* 0 <= source < n else GLB_EINVAL (common.py:68-70) */
  int32_t bins;            /* histogram bins for NS/HP MDT (default 10) */
  int32_t chunked;         /* EP work chunking (edge_based.py:81-85) */
  int64_t mdt;             /* <= 0: compute_mdt(build_histogram(g, bins)) */
  int64_t max_cells;       /* EP COO cell budget (csr.py:16-18) */
  int32_t block_size;      /* KernelConfig.block_size: HP fallback threshold (hierarchical.py:49) */
  int32_t hp_fallback;     /* run_hp(fallback=...) */
  int64_t virtual_threads; /* KernelConfig.virtual_threads (0 = auto); reported only */
  int32_t dist_bits;       /* 0 = auto (24 -> 32 -> 64 on overflow), 24, 32, 64 */
  int32_t loop_mode;       /* GLB_LOOP_HOST / GLB_LOOP_GRAPH */
  int32_t record_timing;   /* per-launch CUDA event timing into records */
  int32_t instrument;      /* 1: record every launch's per-thread work list
                              (MetricsRecord.per_thread_work, engine.py:142-174);
                              fetch with glb_run_thread_work */
} glb_run_params;

typedef struct glb_run_stats {
  int32_t status;          /* GLB_OK or GLB_ECOO_CAPACITY (EP infeasible) */
  int32_t dist_bits;       /* distance width actually used */
  int64_t iterations;      /* super-iterations */
  int64_t launches;        /* relax-kernel invocations (one MetricsRecord each) */
  int64_t sub_iterations;  /* HP sub-iteration launches */
  int64_t relax_ops;       /* atomic_relax_min calls (engine.py:120-139) */
  int64_t push_ops;        /* successful worklist reservations (worklist.py:84-130) */
  int64_t edges_examined;  /* sum of per-thread work */
  int64_t active_items;    /* sum over launches of worklist sizes */
  int64_t mdt;             /* threshold used by NS/HP, else 0 */
  int64_t num_split_nodes; /* NS */
  int64_t num_children;    /* NS */
  double split_fraction;   /* NS split fraction (splitting.py:44-50), else -1 */
  double device_ms;        /* CUDA-event time of the whole run on the library stream */
  double kernel_ms;        /* sum of relax-kernel event times (record_timing=1) */
  double overhead_ms;      /* device time outside relax kernels (scan/split/coo/init) */
  double setup_ms;         /* per-run preprocessing (histogram, split, coo, init) */
  int64_t n_records;       /* records produced (may exceed the caller's capacity) */
} glb_run_stats;

/* One kernel invocation, mirroring MetricsRecord (engine.py:142-174).
 * per_thread_work is summarised on device (sum / sum of squares / max); with
 * glb_run_params.instrument the exact list of the record's `threads` values
 * starts at thread_work_offset of the run's list (glb_run_thread_work; -1 =
 * not recorded). */
typedef struct glb_record {
  int32_t iteration;
  int32_t sub_iteration;   /* -1 = None */
  int32_t tag;             /* GLB_BS..GLB_HP or GLB_TAG_WD_FALLBACK */
  int32_t reserved;
  int64_t active_items;
  int64_t threads;
  int64_t work_total;
  int64_t work_max;
  double work_sumsq;
  int64_t relax_ops;
  int64_t push_ops;
  double kernel_ms;
  double overhead_ms;
  int64_t thread_work_offset;
} glb_record;

/* ---- library / device ---- */
const char* glb_last_error(void);
const char* glb_version(void);
int glb_device_count(int* count);
/* number of CUDA kernels this library has launched in the process */
uint64_t glb_kernel_launches(void);
/* Return the device memory cached by the library's allocator (graph arrays and
 * workspaces of destroyed graphs are kept for reuse) to the driver.
 * device < 0: every device.  *bytes_released may be NULL. */
int glb_release_cached_memory(int device, int64_t* bytes_released);

/* ---- graph (csr.py:42-118) ---- */
/* Copies the host CSR (int64 row_offsets[n+1], col[m], weights[m] or NULL) into
 * HBM on `device`.  Host worker threads validate and narrow col/weights to
 * 32 bits (8 bits for weight chunks that fit) into pinned staging buffers, so
 * PCIe carries the narrow layout.  Validates
 * the CsrGraph invariants (csr.py:66-85); weights must be < 2^32. */
int glb_graph_create(const int64_t* row_offsets, const int64_t* col,
                     const int64_t* weights_or_null, int64_t n, int64_t m,
                     int device, glb_graph** out);
/* R-MAT straight into HBM, draw-for-draw identical to generate_rmat
 * (generators.py:23-58) + CsrGraph.from_edges (csr.py:97-118) under numpy's
 * PCG64: state/inc are default_rng(seed).bit_generator.state (hi, lo words);
 * t_a, t_ab, t_abc are a, a+b, a+b+c as computed by the reference. */
int glb_graph_create_rmat(int scale, int64_t edge_factor, double t_a, double t_ab, double t_abc,
                          const uint64_t* state_hi_lo, const uint64_t* inc_hi_lo, int weighted,
                          int64_t max_weight, int device, glb_graph** out);
/* Device CSR back to host int64 arrays (any pointer may be NULL). */
int glb_graph_download(glb_graph* g, int64_t* row_offsets, int64_t* col, int64_t* weights);
/* The device-native layout back to the host without widening: uint32
 * columns / weights (any pointer may be NULL). */
int glb_graph_download_u32(glb_graph* g, int64_t* row_offsets, uint32_t* col, uint32_t* weights);
int glb_graph_destroy(glb_graph* g);
int glb_graph_info(const glb_graph* g, int64_t* n, int64_t* m, int* weighted,
                   int* device);
/* cudaStream_t of the graph's library stream (for event timing by callers) */
int glb_graph_stream(const glb_graph* g, void** stream);

/* ---- strategies (strategies/__init__.py:17-41) ---- */
/* dist_out: caller-allocated int64[n]; INF is INT64_MAX (engine.py:27).
 * dist_out may be NULL: the distances then stay in HBM (no device->host copy).
 * records may be NULL; *n_records is the capacity on input (ignored when
 * records is NULL) and stats->n_records the produced count on output.
 * EP over the COO budget returns GLB_OK with stats->status = GLB_ECOO_CAPACITY
 * and leaves dist_out untouched (edge_based.py:41-46). */
int glb_run(glb_graph* g, const glb_run_params* params, int64_t* dist_out,
            glb_run_stats* stats, glb_record* records, int64_t records_capacity);

/* Records of the graph's most recent glb_run, from `offset` on (for callers
 * whose capacity was too small); *written receives the count copied. */
int glb_run_records(glb_graph* g, int64_t offset, glb_record* records,
                    int64_t capacity, int64_t* written);

/* Per-thread work of the graph's most recent instrumented glb_run: values
 * [offset, offset + count) of its list (uint32 per launched thread; each
 * record's `threads` values start at its thread_work_offset).  *total (may
 * be NULL) receives the list length. */
int glb_run_thread_work(glb_graph* g, int64_t offset, int64_t count, uint32_t* out,
                        int64_t* total);

/* ---- sharded runs, host-staged exchange: 1-D vertex partition across ranks ----
 * The portable step-by-step form of the peer run below, for transports the
 * caller drives (torch.distributed NCCL / gloo).  Every rank holds the graph over the GLOBAL id space with only its own rows
 * (glb_graph_restrict) and runs BS / WD / HP locally; per iteration:
 *   glb_shard_local  -> run to the iteration boundary, split the improved
 *                       vertices by owner: send_buf (device, u64 entries
 *                       dist << 32 | v) grouped by owner, counts per owner;
 *   (host exchanges the buckets, e.g. NCCL all-to-all)
 *   glb_shard_apply  -> relax the received entries (device buffer);
 *   glb_shard_advance-> swap worklists; *frontier = local frontier size
 *                       (global termination: all-reduce of frontiers);
 *   glb_shard_finish -> int64 distances of the owned range [lo, hi). */
int glb_graph_partition(glb_graph* g, int parts, int64_t* bounds);
int glb_graph_restrict(glb_graph* g, int64_t v_lo, int64_t v_hi);
int glb_shard_begin(glb_graph* g, const glb_run_params* params, const int64_t* bounds,
                    int parts, int rank);
int glb_shard_local(glb_graph* g, int64_t* send_counts, void* send_buf,
                    int64_t send_capacity, int64_t* local_next);
int glb_shard_apply(glb_graph* g, const void* recv_buf, int64_t nrecv);
int glb_shard_advance(glb_graph* g, int64_t* frontier);
int glb_shard_finish(glb_graph* g, int64_t* dist_owned, glb_run_stats* stats);

/* ---- sharded runs over peer memory (the product path) ----
 * The whole BSP loop of a 1-D vertex partition runs inside the library.  Each
 * rank owns an exchange region in its HBM (per-sender inbox segments and
 * mailbox slots, double-buffered by iteration parity); ranks write each
 * other's regions directly with P2P stores over NVLink / NVSwitch -- regions
 * of other processes are mapped with CUDA IPC, ranks of one process use plain
 * device pointers.  One iteration: local relaxation to the iteration boundary
 * (the strategy's loop graph), remote improvements scattered straight into
 * the owners' inboxes, mailbox publish (release), wait for every peer
 * (acquire), relaxation of the received entries, advance; one control-block
 * read-back per iteration carries the global termination and overflow
 * verdicts.  Distance tiers 24 -> 32 -> 64 bits as glb_run, switched on
 * every rank at the same iteration.  Replaces the reference's host loop
 * (node_based.py:33-80, workload.py:175-189, hierarchical.py:54-136) across
 * ranks; strategies BS, WD and HP (others: GLB_EINVAL).
 *
 *   glb_peer_create   exchange region for rank `rank` of `parts` on g's device
 *                     (g: the rank's restricted shard, glb_graph_restrict)
 *   glb_peer_handle   GLB_PEER_HANDLE_BYTES IPC handle of the region
 *   glb_peer_connect  map every other rank's region from the gathered handles
 *                     (parts * GLB_PEER_HANDLE_BYTES, rank order)
 *   glb_peer_connect_local  connect ranks living in this process
 *   glb_peer_run      one rank's whole run (blocking; every rank calls it with
 *                     the same params); int64 distances of the owned range
 *   glb_peer_run_local      every rank of this process, interleaved on one
 *                     host thread (virtual ranks on one GPU, or one process
 *                     driving several GPUs)
 * A peer that never publishes makes the others fail with GLB_ECUDA after
 * GLB_PEER_TIMEOUT_S seconds (default 120) instead of hanging. */
#define GLB_PEER_HANDLE_BYTES 64
#define GLB_PEER_IPC 1    /* regions of other processes mapped via CUDA IPC */
#define GLB_PEER_LOCAL 2  /* all ranks in this process */
typedef struct glb_peer glb_peer;
typedef struct glb_peer_stats {
  int64_t bsp_iterations;  /* exchange rounds (== global iterations) */
  int64_t sent_entries;    /* (dist, v) updates this rank wrote into peers' inboxes */
  int64_t recv_entries;    /* updates it received */
  int32_t entry_bytes;     /* 8 (<= 32-bit distances) or 16 */
  int32_t parts;
  int32_t rank;
  int32_t transport;       /* GLB_PEER_IPC / GLB_PEER_LOCAL */
  double exchange_ms;      /* device time of scatter .. advance, summed over iterations */
  double wait_ms;          /* of which polling for peers */
} glb_peer_stats;
int glb_peer_create(glb_graph* g, const int64_t* bounds, int parts, int rank, glb_peer** out);
int glb_peer_handle(glb_peer* p, void* handle_out);
int glb_peer_connect(glb_peer* p, const void* handles);
int glb_peer_connect_local(glb_peer* const* peers, int parts);
int glb_peer_run(glb_peer* p, const glb_run_params* params, int64_t* dist_owned,
                 glb_run_stats* stats, glb_peer_stats* xstats);
int glb_peer_run_local(glb_peer* const* peers, int parts, const glb_run_params* params,
                       int64_t* const* dist_owned, glb_run_stats* stats, glb_peer_stats* xstats);
int glb_peer_destroy(glb_peer* p);

/* ---- graph files (io.py) ---- */
/* read_csr_bin (io.py:141-170) straight into HBM: the "CSRG" v1 cache is
 * memory-mapped and streamed through glb_graph_create's narrowing upload. */
int glb_graph_load_csrg(const char* path, int device, glb_graph** out);
/* load_dimacs_gr (io.py:26-81, kind 0) / load_edge_list (io.py:84-122, kind 1
 * unweighted, kind 2 weighted), grouped like CsrGraph.from_edges; the int64
 * arrays (row n+1, col m, w m or NULL) are malloc'd by the library: release
 * them with glb_free. */
int glb_read_text_graph(const char* path, int kind, int64_t* n, int64_t* m, int* weighted,
                        int64_t** row, int64_t** col, int64_t** w);
void glb_free(void* p);

/* ---- measurement ---- */
/* Ceilings of the relaxation's memory pattern measured on this graph's own
 * col array (no reference counterpart; used by bench.py's roofline):
 * out4[0] col stream GB/s, out4[1] gathers/s of dist[col[e]] (G/s, 8-byte
 * cells, full occupancy), out4[2] atomicMin(dist[col[e]]) G/s, out4[3] MB of
 * the gathered cell array. */
int glb_measure_gather(glb_graph* g, double* out4);

/* ---- degree analysis (degrees.py) ---- */
int glb_degree_stats(glb_graph* g, int64_t* max_degree, int64_t* sum_degree,
                     double* sum_sq_degree);
/* counts: caller-allocated int64[bins] (1-based bin b at counts[b-1]) */
int glb_histogram(glb_graph* g, int bins, int64_t* counts, int64_t* max_degree,
                  int32_t* arg_max_bin, int64_t* mdt);

/* ---- node splitting (splitting.py:58-99) ----
 * Two-call protocol: call with new_row_offsets == NULL to get *new_n and
 * *num_children; then call again with buffers of int64 [new_n+1], [m], [m]
 * (weights, ignored when unweighted), [num_children], [n+1]. */
int glb_split_graph(glb_graph* g, int64_t mdt, int64_t* new_n,
                    int64_t* num_children, int64_t* new_row_offsets,
                    int64_t* new_col, int64_t* new_weights, int64_t* parent_of,
                    int64_t* children_start);

/* ---- COO expansion (csr.py:155-170) ----
 * Returns GLB_ECOO_CAPACITY when (3 if weighted else 2) * m > max_cells.
 * src_out: int64[m] (dst/weights are the CSR arrays, copied by the caller). */
int glb_csr_to_coo(glb_graph* g, int64_t max_cells, int64_t* src_out);

/* ---- distance certificate (oracles.py:13-82, bench.py:186-196) ----
 * Proves dist (int64[n], INF = INT64_MAX) the exact BFS (algo GLB_BFS) or
 * SSSP (GLB_SSSP) distances from source without an oracle: d[source] == 0,
 * no edge out of a reached node can lower its head (d[v] <= d[u] + w), and
 * every reached node is reachable from the source over tight edges
 * (d[u] + w == d[v]).  n_bad = number of nodes violating a rule (0 = the
 * array is correct), first_bad = the smallest such node id or -1. */
int glb_validate(glb_graph* g, int32_t algo, int64_t source, const int64_t* dist,
                 int64_t* n_bad, int64_t* first_bad);

/* ---- device primitives on host arrays (scan.py, workload.py) ---- */
/* out[i] = values[0] + ... + values[i]; GLB_EOVERFLOW past int64. */
int glb_inclusive_scan(const int64_t* values, int64_t n, int64_t* out, int device);
/* Per-thread (worklist index, edge offset) by binary search of the inclusive
 * prefix (workload.py:45-72); idle threads get node_off = -1, edge_off = 0. */
int glb_find_offsets(const int64_t* prefix, int64_t size, int64_t edges_per_thread,
                     int64_t threads, int64_t* node_off, int64_t* edge_off,
                     int device);

#ifdef __cplusplus
}
#endif

#endif /* GRAPHLB_B200_H */
