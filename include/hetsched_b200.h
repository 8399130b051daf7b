/*
 * hetsched_b200.h — C ABI of the B200-native graph-partition scheduler hot path.
 *
 * The reference (arXiv 1502.07451, package `hetsched`, /root/reference/pkg)
 * has no FFI: its boundary is the Python API re-exported by
 * pkg/src/hetsched/__init__.py:3-12. Every entry point below replaces the
 * compute behind one of those Python functions; the Python package
 * `paper_1502_07451_b200` keeps the reference names and signatures and calls
 * these through ctypes (see INTEGRATION.md for the binding).
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors) unless the name ends in `_host`. The caller owns every buffer;
 *    the library only allocates stream-ordered scratch (cudaMallocAsync).
 *  - `stream` is a cudaStream_t passed as void*. Calls are asynchronous
 *    unless documented otherwise; results are valid after the stream syncs.
 *  - Return value: 0 (HS_OK) or a negative HS_E* status. The message of the
 *    last failure on the calling thread is in hs_last_error().
 *  - Node index space: a DAG's nodes are the reference's node ids sorted
 *    ascending, numbered 0..n-1; `root` is the index of the SOURCE node.
 *    "Kernel" index space: the n-1 non-root nodes in ascending id order
 *    (the reference's graph.kernel_ids(), graph.py:92-94).
 *  - Two-way part ids: 0 = CPU, 1 = GPU (METIS partition-file convention,
 *    graphio.py:328). k-way part ids: 0..k-1.
 *  - Floating point: fp64 everywhere; kernels on the bit-exact paths are
 *    compiled without FMA contraction.
 */
#ifndef HETSCHED_B200_H
#define HETSCHED_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_OK 0
#define HS_EINVAL (-1)      /* bad argument (sizes, null pointers) */
#define HS_ECUDA (-2)       /* CUDA runtime error */
#define HS_ELIMIT (-3)      /* size beyond a documented limit */
#define HS_EPOLICY (-4)     /* unknown policy id */
#define HS_EDEADLOCK (-5)   /* simulation could not finish every node */
#define HS_EPARTITION (-6)  /* partition precondition failed (zero weight, ...) */

/* Directed task DAG, device CSR. Edges are stored once, sorted by
 * (src, dst) — the reference's sorted(graph.edges) order (graph.py:114,
 * partition.py:53). */
typedef struct hs_dag {
    int32_t n;               /* nodes, including the root */
    int32_t root;            /* index of the SOURCE node */
    int64_t m;               /* edges */
    const int64_t *out_ptr;  /* [n+1] */
    const int32_t *out_dst;  /* [m]   sorted by (src, dst) */
    const int64_t *in_ptr;   /* [n+1] */
    const int32_t *in_src;   /* [m]   per dst, ascending src (graph.py:89-90) */
    const int32_t *in_eid;   /* [m]   edge index (out order) of each in-entry */
    const double *w_cpu;     /* [n] */
    const double *w_gpu;     /* [n] */
    const double *w_xfer;    /* [m] out order */
    const int64_t *bytes;    /* [m] out order */
} hs_dag_t;

/* A batch of independent DAGs packed back to back (config 5: one graph per
 * simulation). Graph b owns nodes [node_off[b], node_off[b+1]) and edges
 * [edge_off[b], edge_off[b+1]); indices inside the arrays are LOCAL to the
 * graph (0..n_b-1 / 0..m_b-1); out_ptr/in_ptr are local too and have
 * n_b+1 entries starting at node_off[b]+b. */
typedef struct hs_dag_batch {
    int32_t batch;
    int64_t total_nodes;         /* node_off[batch] */
    int64_t total_edges;         /* edge_off[batch] */
    const int64_t *node_off;     /* [batch+1] */
    const int64_t *edge_off;     /* [batch+1] */
    const int32_t *root;         /* [batch] local root index */
    const int64_t *out_ptr;      /* [node_off[batch] + batch] */
    const int32_t *out_dst;
    const int64_t *in_ptr;
    const int32_t *in_src;
    const int32_t *in_eid;
    const double *w_cpu;
    const double *w_gpu;
    const double *w_xfer;
    const int64_t *bytes;
} hs_dag_batch_t;

/* Undirected weighted graph over the kernels (root excluded), device CSR —
 * the graph `fm_refine` builds (partition.py:153-158) and `emit_metis`
 * exports (graphio.py:285-304). For the exact 2-way path the neighbour order
 * of each vertex is the reference's (sorted-edge order); the k-way path is
 * order-independent. */
typedef struct hs_ugraph {
    int32_t n;               /* vertices (kernels) */
    int64_t nnz;             /* adjacency entries = 2 * undirected edges */
    const int64_t *xadj;     /* [n+1] */
    const int32_t *adjncy;   /* [nnz] */
    const double *adjwgt;    /* [nnz] fp64 edge weights (exact 2-way path) */
    const int32_t *adjwgt_i; /* [nnz] integer edge weights (k-way path);
                                NULL = every edge weighs 1 (METIS adjwgt = NULL) */
    const double *vwgt;      /* [n]  fp64 vertex weights (exact 2-way path) */
    const int32_t *vwgt_i;   /* [n]  integer vertex weights (k-way path);
                                total must be < 2^31 */
    const int32_t *twin;     /* [nnz] optional: position of the reverse entry
                                (u in v's list <-> v in u's list); enables the
                                ghost-part refinement on the finest level */
} hs_ugraph_t;

/* ---- status / library ------------------------------------------------ */
const char *hs_last_error(void);
const char *hs_version(void);
/* Number of launches of this library's kernels since load (evidence for the
 * bench's gpu_launches field). */
int64_t hs_launch_count(void);
/* Live kernel profiling: when enabled, designated launches are bracketed by
 * CUDA events on their stream and booked as (launches, device ms,
 * algorithmic bytes) per kernel name. hs_profile_report writes
 * "name,launches,ms,bytes\n" lines (synchronises the pending events) and
 * returns the full text length. */
void hs_profile_enable(int on);
void hs_profile_reset(void);
int hs_profile_report(char *buf, int len);

/* ---- K0 exact sums (fsum) --------------------------------------------
 * Replaces math.fsum in total_weights (graph.py:327-332) and
 * workload_ratio (costs.py:239-253): out_host[0..2] = correctly rounded
 * sums of w_cpu, w_gpu over nodes (root skipped unless include_root) and
 * of w_xfer over all edges. Synchronous. */
int hs_exact_totals(const hs_dag_t *g, int include_root, double *out_host, void *stream);
/* Per graph of a batch: out[3b..3b+2] (device) = fsum of w_cpu, w_gpu, w_xfer. */
int hs_exact_totals_batch(const hs_dag_batch_t *g, int include_root, double *out, void *stream);

/* ---- K2 evaluate -------------------------------------------------------
 * Replaces partition.evaluate / _finish (partition.py:60-84) for `batch`
 * two-way assignments of one DAG. part: [batch][n_kernels] int8 (0 CPU /
 * 1 GPU). Per assignment: cut = Σ w_xfer over inter-kernel edges with
 * different sides, cpu_w = Σ node weight on CPU, total = Σ node weight.
 * mode 0: sums in the reference's sequential order (bit-exact with the
 *         reference's builtin sum) — one thread per assignment;
 * mode 1: correctly rounded sums (superaccumulator), fully parallel.
 * weight_source: 0 = CPU weights, 1 = GPU weights (partition.py:48-49).
 * out: cut[batch], cpu_w[batch], total[batch] (device). */
int hs_evaluate2(const hs_dag_t *g, const int8_t *part, int32_t batch,
                 int weight_source, int mode,
                 double *cut, double *cpu_w, double *total, void *stream);

/* k-way batched evaluation on the directed DAG (config 2): for each of
 * `batch` assignments part[b][n] (int32, node index space, root's entry
 * ignored) computes the integer edge cut over inter-kernel edges
 * (cut_bytes: Σ bytes, cut_edges: count), per-part loads in int64 (from
 * vwgt_i, [batch][k]) and the distinct-producer transfer count/bytes: one
 * transfer per (producer u, consumer part p != part[u]) pair — the
 * k-memory-node generalisation of the simulator's item dedup
 * (sim.py:86-89,141-144); its bytes are those of u's first edge into p. */
int hs_evaluate_kway(const hs_dag_t *g, const int32_t *part, int32_t batch, int32_t k,
                     const int64_t *vwgt_i, int64_t *cut_bytes, int64_t *cut_edges,
                     int64_t *loads, int64_t *xfer_count, int64_t *xfer_bytes,
                     void *stream);

/* ---- K7 levels / critical path ----------------------------------------
 * level[n]: longest-path depth in edges from the root (root = 0).
 * finish[n]: longest path with node duration min(w_cpu, w_gpu) and zero
 * transfer cost — critical_path_lower_bound (sim.py:239-247); *cp_host =
 * max(finish) (synchronous). mode 0 = min(cpu,gpu) durations; mode 1 =
 * w_gpu only; mode 2 = w_cpu only. n_levels_host receives max level + 1. */
int hs_levels(const hs_dag_t *g, int mode, int32_t *level, double *finish,
              double *cp_host, int32_t *n_levels_host, void *stream);

/* Device validation (validate, graph.py:113-150) of the checks a CSR can
 * violate. counts_host[7] = offenders per check, first_host[7] = smallest
 * offending index (-1 if none): 0 node with a negative weight, 1 root with
 * non-zero weights, 2 self-loop edge, 3 edge with negative transfer weight,
 * 4 edge with negative byte count, 5 node never released by Kahn's algorithm
 * with self-loops ignored (first = the reference's CycleError member,
 * graph.py:153-172), 6 non-root node without predecessors. node_bad [n] /
 * edge_bad [m] (optional, device int8) receive per-item bit masks (node:
 * 1 negative, 2 root weight, 4 no predecessor, 8 on/after a cycle; edge:
 * 1 self-loop, 2 negative transfer, 4 negative bytes). Synchronous. The
 * object-model checks (duplicate ids/edges, unknown endpoints, root kind)
 * stay on the host. */
int hs_validate_dag(const hs_dag_t *g, int64_t *counts_host, int32_t *first_host,
                    int8_t *node_bad, int8_t *edge_bad, void *stream);

/* Level-synchronous makespan of a given assignment:
 * finish[v] = max over in-edges (finish[u] + w_xfer(u,v) if the edge crosses)
 * + (dev[part[v]] ? w_gpu[v] : w_cpu[v]); an edge crosses when part[u] !=
 * part[v], or, from the root (data in host memory), when v's part is a GPU
 * part. part: [n] int32 in [0, k) (root entry ignored); dev: [k] int8 (0 CPU,
 * 1 GPU). makespan_host = max finish — the infinite-workers lower bound of
 * the schedule the assignment induces (sim.py:239-247 with transfers).
 * fp64 max/add once per node: order-independent, bit-exact. */
int hs_assigned_makespan(const hs_dag_t *g, const int32_t *part, const int8_t *dev, int32_t k,
                         int32_t *level, double *finish, double *makespan_host, void *stream);

/* topological_order (graph.py:153-172): the lexicographically smallest
 * topological order (Kahn with an id min-heap, self-loops ignored), bit for
 * bit. order[n] receives node indices; *count_host = nodes output (n unless
 * there is a cycle); on a cycle *stuck_host = the smallest index never
 * released (the reference's CycleError member), else -1. *rounds_host
 * (optional): batched rounds used (0 = the identity fast path: every edge
 * points to a larger index). Synchronous. */
int hs_topological_order(const hs_dag_t *g, int32_t *order, int32_t *count_host,
                         int32_t *stuck_host, int32_t *rounds_host, void *stream);

/* Level order: nodes sorted by (level, index) — order[n]. */
int hs_level_order(const hs_dag_t *g, const int32_t *level, int32_t n_levels,
                   int32_t *order, void *stream);

/* ---- vertex orders for the k-way band start (csrc/order.cu) -----------
 * The partitioner's band start cuts kernel positions into weight ranges; it
 * relies on positions following the DAG's layers, as creation-order numbering
 * does (every edge u -> v with u < v). Other numberings are relabelled in
 * longest-path level order (ties by position) first.
 *
 * result_host = 1 when every non-root edge u -> v has u < v (first entry of
 * each sorted out-list checked). */
int hs_dag_is_topological(const hs_dag_t *g, int32_t *result_host, void *stream);
/* Kernel positions (root excluded) stably sorted by level (hs_levels):
 * perm[new] = old position, inv[old] = new position; both [n-1]. */
int hs_level_permutation(const hs_dag_t *g, const int32_t *level, int32_t n_levels,
                         int32_t *perm, int32_t *inv, void *stream);
/* The kernel graph relabelled: row i of the output is row perm[i] of g with
 * every neighbour id u replaced by inv[u]; vwgt_i permuted alike. Output
 * arrays: xadj [n+1], adjncy/adjwgt_i [nnz] (adjwgt_i only when g has
 * integer weights), vwgt_i [n]. */
int hs_ugraph_permute(const hs_ugraph_t *g, const int32_t *perm, const int32_t *inv,
                      int64_t *xadj, int32_t *adjncy, int32_t *adjwgt_i, int32_t *vwgt_i,
                      void *stream);
/* part[perm[i]] = part_new[i] for i < n. */
int hs_parts_unpermute(int32_t n, const int32_t *perm, const int32_t *part_new, int32_t *part,
                       void *stream);

/* ---- K8 batched discrete-event simulation -----------------------------
 * Replaces sim.simulate (sim.py:68-204) with EagerPolicy / DmdaPolicy /
 * GraphPartitionPolicy (policies.py:19-99), one simulation per thread,
 * bit-exact (fp64 add/max only, reference event order).
 * policy: 0 eager, 1 dmda, 2 gp (pin[] required: node-index space,
 * 0 CPU / 1 GPU, root entry ignored).
 * Outputs per simulation: makespan, transfer_count, transfer_bytes,
 * busy[2] (CPU, GPU ms), kpd[2] (kernels per device), status (0 ok,
 * HS_EDEADLOCK). If ev != NULL, events are written to ev at offset
 * ev_off[b] (capacity ev_off[b+1]-ev_off[b], >= 2*n_b + 2*m_b) and ev_count[b]
 * receives the number written, in generation order (the caller sorts). */
typedef struct hs_event {
    double time;
    int32_t kind;      /* 0 xfer_start, 1 xfer_end, 2 kernel_start, 3 kernel_end */
    int32_t a;         /* kernel local index, or producer local index (item) */
    int32_t b;         /* item consumer local index for root items, else -1 */
    int32_t resource;  /* worker id, or -1 for the bus */
} hs_event_t;

int hs_simulate_batch(const hs_dag_batch_t *g, int policy, const int8_t *pin,
                      int32_t cpu_workers, int32_t gpu_workers,
                      double *makespan, int64_t *transfer_count, int64_t *transfer_bytes,
                      double *busy, int64_t *kpd, int32_t *status,
                      hs_event_t *ev, const int64_t *ev_off, int64_t *ev_count,
                      void *stream);

/* ---- weight attachment (attach_weights, graph.py:308-324) -------------
 * One entry per distinct (kind, size) pair: form 0 = the value pair cpu/gpu
 * (read from the cost model on the host once), 1 = synthetic MA closed form
 * (ma_cpu * s^2, ma_gpu * s^2 + launch_ms), 2 = synthetic MM (s^3),
 * 3 = zero weights (SOURCE kind / the root), -1 = no cost entry. Device
 * pointers. Transfers: latency_ms + bytes / bandwidth (costs.py:52-55). */
typedef struct hs_cost_table {
    int32_t n_pairs;
    const int32_t *form;   /* [n_pairs] */
    const double *cpu;     /* [n_pairs] (form 0) */
    const double *gpu;     /* [n_pairs] (form 0) */
    double ma_cpu, ma_gpu, mm_cpu, mm_gpu, launch_ms;
    double latency_ms, bandwidth;
} hs_cost_table_t;
/* w_cpu/w_gpu [n] from pair[n] (entry index) and size[n]; w_xfer[m] from
 * bytes[m], or copied from xfer_tab[m] when given (custom transfer models).
 * rank[n] (optional) orders nodes for the error report: *bad_node_host =
 * the smallest rank among nodes without a cost entry (-1 if none);
 * *bad_edge_host = the first edge with a negative byte count (-1 if none).
 * Synchronous. */
int hs_attach_weights(const hs_cost_table_t *t, int32_t n, const int32_t *pair,
                      const int64_t *size, const int32_t *rank, double *w_cpu, double *w_gpu,
                      int64_t m, const int64_t *bytes, const double *xfer_tab, double *w_xfer,
                      int32_t *bad_node_host, int64_t *bad_edge_host, void *stream);

/* Trace products (sim.py:200-236) from a device event buffer of one
 * simulation (count events, node indices local to the graph):
 * hs_trace_sort writes perm[count] = event indices in the reference's order
 * (time, xfer_start < xfer_end < kernel_start < kernel_end, subject as a
 * string with node ids ids[n] (int64), resource name as a string given by
 * res_rank[resource + 1] = rank of the name in string order, bus = -1).
 * hs_trace_metrics: metrics(trace) over the sorted events: out_host[6] =
 * makespan, transfer count, busy CPU ms, busy GPU ms (fp64 sums in event
 * order), kernels on CPU, kernels on GPU; workers [0, cpu_workers) are CPU.
 * Both synchronous. */
int hs_trace_sort(const hs_event_t *ev, int64_t count, const int64_t *ids,
                  const int32_t *res_rank, int32_t *perm, void *stream);
int hs_trace_metrics(const hs_event_t *ev, const int32_t *perm, int64_t count, int32_t n_nodes,
                     int32_t cpu_workers, double *out_host, void *stream);

/* ---- K5/K6 exact two-way partitioner ----------------------------------
 * Replaces partition_heuristic's restart loop + fm_refine
 * (partition.py:137-295) with the reference's exact semantics: one CTA per
 * start order runs _greedy_init -> _repair_balance -> fm_refine; moves,
 * gains, prefix selection and fp64 rounding follow the reference exactly.
 * orders: [n_orders][g->n] kernel positions. If start != NULL the greedy
 * init and repair are skipped and every CTA refines start[n] (fm_refine).
 * Outputs per order: assign[n_orders][n] (0 CPU/1 GPU), cut, err.
 * weights: [n] node weights (the configured source), w_total = their
 * builtin sum (host-computed in id order). */
int hs_fm2(const hs_ugraph_t *g, const double *edge_w_sorted,
           const int32_t *edge_u, const int32_t *edge_v, int64_t n_edges,
           const double *weights, double r_cpu, double tol,
           const int32_t *orders, int32_t n_orders, const int8_t *start,
           int8_t *assign, double *cut, double *err, void *stream);

/* Batched hs_fm2 for G independent graphs (config 5's gp policy builds): one
 * CTA per (graph, start order). Arrays are concatenated: node_off/adj_off/
 * edge_off [G+1] give each graph's slice of the kernel-indexed arrays
 * (weights, assignment rows), of adjncy/adjwgt and of the edge list; xadj
 * holds n_g + 1 LOCAL offsets per graph; orders/assign are [G][R][n_g] at
 * R * node_off[g]; cut/err/status are [G][R]. r_cpu: [G] device. */
int hs_fm2_batch(int32_t G, const int64_t *node_off, const int64_t *adj_off,
                 const int64_t *edge_off, int64_t total_nodes, int32_t max_n,
                 const int64_t *xadj, const int32_t *adjncy, const double *adjwgt,
                 const double *edge_w, const int32_t *edge_u, const int32_t *edge_v,
                 const double *weights, const double *r_cpu, double tol,
                 const int32_t *orders, int32_t n_orders, int8_t *assign, double *cut,
                 double *err, int32_t *status, void *stream);

/* gp_build for every graph of a batch (policies.py:102-108) as the DES pin
 * array: pin[node] = 1 when the graph's gp partition puts the kernel on the
 * GPU (root 0). Workload ratios from the fsum totals, the reference's start
 * orders (stable descending weight, then `restarts` shuffles [restarts][n]
 * drawn on the host with the reference's random.Random — every graph must
 * have n_shuffle kernels), hs_fm2_batch, the reference's winner key.
 * flags_host[G]: per graph 1 no kernels, 2 zero total time, 4 zero kernel
 * weight (nothing is partitioned when any flag is set). Synchronous. */
int hs_gp_pins_batch(const hs_dag_batch_t *g, int32_t restarts, const int32_t *shuffles,
                     int32_t n_shuffle, double tol, int8_t *pin, int32_t *flags_host,
                     void *stream);

/* Exhaustive 2-way oracle (brute_force_partition, partition.py:87-134) on
 * the device for n <= 30 (the Python API keeps the reference's limit of 20).
 * Writes the winning mask (bit n-1-k set = kernel k on GPU) to *mask_host
 * and whether it is feasible. Synchronous. */
int hs_brute2(int32_t n, const double *weights, double r_cpu, double tol,
              const int32_t *edge_a, const int32_t *edge_b, const double *edge_w,
              int64_t n_edges, int64_t *mask_host, int32_t *feasible_host, void *stream);

/* ---- K1/K3/K4/K5/K6 multilevel k-way partitioner -----------------------
 * Balanced min-cut k-way partition of the undirected integer-weighted
 * graph (METIS_PartGraphKway's role): heavy-edge
 * matching, contraction, parallel initial partitioning on the coarsest
 * graph, projection and boundary refinement per level. Balance: for every
 * part p, |w_p/total - tpwgts[p]| <= tol (SURVEY App. B k-way
 * generalisation of partition.py:72). tpwgts_host: [k] host fractions.
 * part: [n] int32 output. stats_host (optional, 8 entries): cut (integer,
 * each undirected edge once), levels, coarsest n, max |w_p/total - t_p| *
 * 1e9, feasible, refinement passes, internal weight divisor, 0.
 * If the total edge weight reaches 2^30 the partitioner works on weights
 * divided by a common factor (min 1); the reported cut uses the originals. */
int hs_partition_kway(const hs_ugraph_t *g, int32_t k, const double *tpwgts_host,
                      double tol, uint64_t seed, int32_t *part, int64_t *stats_host,
                      void *stream);

/* hs_partition_kway plus caller-supplied start partitions of the finest
 * graph (device int32 [n_starts][n], values in 0..k-1; n <= 4096): each start
 * is FM-refined with the partitioner's own candidates and competes under the
 * same (balance violation, cut) ranking, so the result is never worse than
 * the best start refined. The Python layer passes the reference heuristic's
 * recursive 2-way partition here (partition.py:258-295). */
int hs_partition_kway_starts(const hs_ugraph_t *g, int32_t k, const double *tpwgts_host,
                             double tol, uint64_t seed, const int32_t *starts, int32_t n_starts,
                             int32_t *part, int64_t *stats_host, void *stream);

/* METIS_PartGraphKway-compatible front end (idx_t = int32, real_t = float,
 * HOST arrays, ncon = 1): the paper's partitioning tool boundary
 * (graphio.py:277-304). Exported twice: under METIS's own
 * name (a METIS caller relinks against this library unchanged) and with the
 * hs_ prefix. Returns METIS's codes: METIS_OK = 1, METIS_ERROR_INPUT = -2,
 * METIS_ERROR_MEMORY = -3, METIS_ERROR = -4 (message in hs_last_error()).
 * Balance: ubvec[0] (default 1.03, or 1 + options[METIS_OPTION_UFACTOR]/1000)
 * becomes tol = (ubvec - 1) * min_p tpwgts[p] in the |w_p/W - t_p| <= tol
 * sense. Honoured options: SEED (8), UFACTOR (16), NUMBERING (17; 1 =
 * 1-based xadj/adjncy/part). objval = edge cut. Synchronous, default stream. */
int METIS_PartGraphKway(const int32_t *nvtxs, const int32_t *ncon, const int32_t *xadj,
                        const int32_t *adjncy, const int32_t *vwgt, const int32_t *vsize,
                        const int32_t *adjwgt, const int32_t *nparts, const float *tpwgts,
                        const float *ubvec, const int32_t *options, int32_t *objval,
                        int32_t *part);
int hs_METIS_PartGraphKway(const int32_t *nvtxs, const int32_t *ncon, const int32_t *xadj,
                           const int32_t *adjncy, const int32_t *vwgt, const int32_t *vsize,
                           const int32_t *adjwgt, const int32_t *nparts, const float *tpwgts,
                           const float *ubvec, const int32_t *options, int32_t *objval,
                           int32_t *part);

/* Symmetrise a DAG into the kernel-space undirected graph used by
 * hs_partition_kway (K1): root and root edges dropped, vertex v (kernel
 * position) adjacent to every predecessor and successor, adjwgt_i from
 * edge_w_i (out order), vwgt_i copied from node_w_i (node index space).
 * edge_w_i_in (optional) holds the same weights in in-order (the DAG's CSC
 * copy of the edge attribute); without it they are gathered via in_eid.
 * twin (optional, [2m] int32) receives each entry's reverse-entry position. 
 * xadj/adjncy/adjwgt_i/vwgt_i are caller buffers sized (n-1)+1 / 2m.
 * adjwgt_i == NULL writes no edge weights (the caller found them uniform with
 * hs_int32_stats and partitions with adjwgt_i = NULL, i.e. unit weights as in
 * METIS's adjwgt = NULL, scaling the cut by the common weight); edge_w_i may
 * then be NULL too. */
int hs_symmetrize(const hs_dag_t *g, const int32_t *edge_w_i, const int32_t *edge_w_i_in,
                  const int32_t *node_w_i, int64_t *xadj, int32_t *adjncy, int32_t *adjwgt_i,
                  int32_t *vwgt_i, int32_t *twin, int64_t *nnz_host, void *stream);
/* The rows of kernel positions [kv0, kv1) only (one rank's shard): xadj has
 * kv1-kv0+1 entries starting at 0, adjncy holds GLOBAL kernel positions,
 * vwgt_i[i] is the weight of kernel kv0+i. twin must be NULL unless the range
 * is the whole graph. */
int hs_symmetrize_range(const hs_dag_t *g, int32_t kv0, int32_t kv1, const int32_t *edge_w_i,
                        const int32_t *edge_w_i_in, const int32_t *node_w_i, int64_t *xadj,
                        int32_t *adjncy, int32_t *adjwgt_i, int32_t *vwgt_i, int32_t *twin,
                        int64_t *nnz_host, void *stream);

/* In-CSR of a DAG from its out-CSR, on the device: in_ptr [n+1], in_src /
 * in_eid [m] in the reference's in_edges order (per destination, ascending
 * source, graph.py:89-90; in_eid = the edge's out-order index). Replaces the
 * host-side construction of the second half of hs_dag_t, so a caller ships
 * only out_ptr/out_dst. Deterministic. m < 2^31. */
int hs_dag_transpose(int32_t n, int64_t m, const int64_t *out_ptr, const int32_t *out_dst,
                     int64_t *in_ptr, int32_t *in_src, int32_t *in_eid, void *stream);

/* Sum, minimum and maximum of n int32 values on the device (one pass; the
 * uniform-weight test before K1). Synchronous on stream. */
int hs_int32_stats(const int32_t *w, int64_t n, int64_t *sum_min_max_host, void *stream);

/* METIS integer weights of n fp64 weights, elementwise on the device (one
 * pass): out[i] = max(1, floor(w[i] * scale + 0.5)) with the reference's two
 * fp64 roundings (graphio.py:272-274, _scaled), saturated at INT32_MAX (NaN
 * maps to 1). Asynchronous on stream. */
int hs_integer_weights(const double *w, int64_t n, int32_t scale, int32_t *out, void *stream);

/* ---- sharded k-way partition (config 4 at 2/4/8 GPUs) ---------------------
 * One call per rank, all ranks concurrently (one process per GPU, or one host
 * thread per rank in loopback mode on a single GPU). Rank r passes the rows
 * of its contiguous vertex range [v0, v0 + g->n) (hs_symmetrize_range) with
 * global neighbour ids. Ranks exchange through `arena[q]`: one whole device
 * allocation per rank (hs_ipc_alloc; peers' arenas CUDA-IPC mapped, or plain
 * pointers on one GPU), at least hs_kway_dist_arena_bytes(n_global) bytes,
 * zeroed once before the group's first call (epochs persist across calls).
 * Per-vertex state neighbours read (parts, refinement state, fine->coarse
 * maps) is replicated by producer-side peer stores; sums/maxima go through an
 * in-kernel all-reduce over the arenas (integer, rank order: bit-identical on
 * every rank). part_out: [n_global] int32, the whole partition, on every
 * rank. stats_host: as hs_partition_kway (global values). The result is a
 * pure function of (graph, ranges, k, targets, tol, seed). A peer that never
 * arrives makes the call fail with HS_EDEADLOCK after a 30 s watchdog. */
typedef struct hs_dist {
    int32_t rank, size;      /* size <= 8 */
    void *arena[8];          /* arena of every rank, valid on this rank's device */
    int64_t arena_bytes;
    int32_t mode;            /* 0: one process per rank (in-kernel flag barriers);
                                1: ranks are host threads of this process sharing
                                one GPU (loopback: host barriers between phases) */
} hs_dist_t;

int64_t hs_kway_dist_arena_bytes(int32_t n_global);
int hs_partition_kway_dist(const hs_ugraph_t *g_local, int32_t v0, int32_t n_global,
                           const hs_dist_t *dist, int32_t k, const double *tpwgts_host,
                           double tol, uint64_t seed, int32_t *part_out, int64_t *stats_host,
                           void *stream);

/* Device generator of the layered fan-in DAG family of configs 2 and 4:
 * n kernels over ceil(sqrt(n)) layers, m inter-kernel edges spread as evenly
 * as possible over the kernels past layer 0, predecessors drawn uniformly
 * without replacement from all earlier layers by a counter-based RNG
 * (splitmix64 of (seed, node, draw)), root edge to every layer-0 kernel.
 * Writes the full DAG CSR (n+1 nodes incl. root at index 0) into caller
 * buffers sized from hs_layered_sizes(). */
int hs_layered_sizes(int64_t n_kernels, int64_t m_inter, int64_t *n_nodes_host,
                     int64_t *n_edges_host);
int hs_layered_generate(int64_t n_kernels, int64_t m_inter, uint64_t seed,
                        int64_t *out_ptr, int32_t *out_dst, int64_t *in_ptr,
                        int32_t *in_src, int32_t *in_eid, int32_t *layer_of,
                        void *stream);

/* ---- K9 tiled-Cholesky execution (fp64) ------------------------------------
 * No reference counterpart (the reference simulates this DAG, sim.py:135-164).
 * hs_chol_pack: row-major n x n <-> tiles of b x b (b = 512), tile (i, j),
 * i >= j, contiguous row-major at tiles + (i*T + j)*b*b; unpacking zeroes the
 * strictly upper part of the diagonal tiles.
 * hs_chol_execute: runs the task DAG (gen.cholesky_tasks order; kind 0
 * POTRF, 1 TRSM, 2 SYRK, 3 GEMM; tile coordinates ti/tj/tk; successor CSR;
 * in-degree) as one persistent kernel of grid_ctas CTAs (0 = one per SM).
 * dinv: T*4 inverted 128x128 diagonal blocks (scratch, T*4*128*128 doubles).
 * *fail_host != 0 if a pivot was not positive (matrix not SPD). */
int hs_chol_pack(double *A, int32_t n, int32_t b, double *tiles, int32_t to_tiles, void *stream);
int hs_chol_execute(double *tiles, double *dinv, int32_t T, int32_t n_tasks, const int8_t *kind,
                    const int16_t *ti, const int16_t *tj, const int16_t *tk,
                    const int64_t *succ_ptr, const int32_t *succ, const int32_t *indeg,
                    int32_t grid_ctas, int32_t *fail_host, void *stream);
/* Same, with optional device counters (16 x u64, zeroed by the caller):
 * [2*kind] SM cycles spent in items of that kind, [2*kind+1] items run,
 * [8..10] POTRF phases (block updates, 128x128 diagonal factor+inverse,
 * panel solve). */
int hs_chol_execute_stats(double *tiles, double *dinv, int32_t T, int32_t n_tasks,
                          const int8_t *kind, const int16_t *ti, const int16_t *tj,
                          const int16_t *tk, const int64_t *succ_ptr, const int32_t *succ,
                          const int32_t *indeg, int32_t grid_ctas, int32_t *fail_host,
                          unsigned long long *stats, void *stream);

/* Partitioned execution over nranks GPUs (or nranks executors on one GPU):
 * rank r runs the tasks with owner[t] == r. When a task's last work item
 * finishes, its CTA stores the task's output tile (and Dinv[k] for POTRF)
 * into tiles[q]/dinv[q] of every rank q owning a successor — one copy per
 * (producer, destination), the k-node generalisation of the simulator's
 * item dedup (sim.py:86-89,141-144) — then appends the task id to q's inbox
 * ring (system-scope atomics). Idle CTAs drain their own inbox and release
 * local successors. All pointers are device pointers valid on the calling
 * rank's device: peers' buffers are CUDA-IPC mappings (hs_ipc_*) or, for
 * loopback executors, plain pointers on the same device.
 * inbox[r]: n_tasks int64 filled with -1; ctl[r]: 2 uint64 zeroed
 * (tail, head). copies_dev (optional, device u64, caller-zeroed) counts the
 * tiles this rank sent. fail_host != NULL makes the call synchronous (status
 * check); pass NULL when several executors must be launched concurrently. */
typedef struct hs_chol_peers {
    int32_t rank, nranks;               /* nranks <= 8 */
    const int8_t *owner;                /* [n_tasks] */
    double *tiles[8];
    double *dinv[8];
    long long *inbox[8];
    unsigned long long *ctl[8];
} hs_chol_peers_t;

int hs_chol_execute_part(double *tiles, double *dinv, int32_t T, int32_t n_tasks,
                         const int8_t *kind, const int16_t *ti, const int16_t *tj,
                         const int16_t *tk, const int64_t *succ_ptr, const int32_t *succ,
                         const int32_t *indeg, const hs_chol_peers_t *peers, int32_t grid_ctas,
                         int32_t *fail_host, unsigned long long *stats,
                         unsigned long long *copies_dev, void *stream);

/* CUDA IPC plumbing for one-process-per-GPU runs (64-byte opaque handles).
 * Shared buffers must be whole allocations (hs_ipc_alloc): a handle names an
 * allocation base. The executor's watchdog returns HS_EDEADLOCK instead of
 * spinning forever if a peer never delivers a dependency. */
int hs_ipc_alloc(int64_t bytes, void **dev_ptr);
int hs_ipc_free(void *dev_ptr);
int hs_memset_async(void *dev_ptr, int32_t byte_value, int64_t bytes, void *stream);
int hs_ipc_handle(void *dev_ptr, char *handle64);
int hs_ipc_open(const char *handle64, void **dev_ptr);
int hs_ipc_close(void *dev_ptr);

/* ---- DOT ingestion (replaces parse_dot, graphio.py:79-199) ---------------
 * hs_dot_parse parses the UTF-8 bytes text[len] (DEVICE memory) with the
 * reference's DOT subset. A text the reference rejects returns HS_OK with
 * info->status = the DotParseError kind (1 expected a digraph header, got
 * {line!r}; 2 undirected graphs are not supported; 3 cannot parse statement
 * {stmt!r}; 4 bad attribute syntax near {text[pos:pos+20]!r}; 5 no digraph
 * found; 6 missing closing brace), info->err_line its 1-based line and
 * err_a/err_b/err_c byte offsets into text (1: the stripped line [a, b);
 * 3: the statement [a, b); 4: the attribute text [a, b) and the failing
 * position c), and *handle = NULL. Otherwise *handle holds the parse:
 *   names in order of first appearance with their ids (graphio.py:145-158),
 *   the last kind/size/weight_cpu/weight_gpu of each (size via int(float())),
 *   edge declarations in order with bytes/weight_xfer, every attribute's key
 *   and value spans, class (0 kind, 1 size, 2 weight_cpu, 3 weight_gpu,
 *   4 bytes, 5 weight_xfer, 6 style, 7 other) and owner (name rank >= 0, or
 *   -1 - edge index);
 *   info->conv_err = (order << 3) | kind of the first float()/int() failure
 *   in the reference's evaluation order (order = 3 * rank + {0 size, 1
 *   weight_cpu, 2 weight_gpu}, then 3 * n_names + 2 * edge + {0 bytes,
 *   1 weight_xfer}; kind 1 ValueError, 2 int(inf), 3 int(nan)), -1 if none;
 *   info->n_slow literals listed as (order, attribute) for the caller to
 *   convert: int(float()) values beyond int64 (Python ints) and exponents
 *   beyond +-100000 with more than 19 significant digits.
 * hs_dot_fetch copies the parse to caller HOST arrays (any may be NULL);
 * hs_dot_csr_size / hs_dot_csr build the device CSR of the graph TaskGraph
 * would hold (ids ascending, edges by (src, dst), a later duplicate edge
 * wins, the synthesized root and its edges when no SOURCE node exists);
 * hs_dot_release frees the handle. */
typedef struct hs_dot_info {
    int32_t status, err_line, err_a, err_b, err_c;
    int32_t name_b, name_e;      /* digraph name group [b, e), b < 0: none */
    int32_t n_names, n_edges, n_attrs, n_slow;
    int32_t root_rank;           /* first name of kind SOURCE, -1: none */
    int64_t conv_err;
    int64_t max_id;              /* the largest assigned id */
} hs_dot_info_t;

typedef struct hs_dot_host {
    int64_t *id; int32_t *kind_attr; uint64_t *kind_hash; int64_t *size;
    double *w_cpu, *w_gpu; uint8_t *has_pred;                 /* [n_names] */
    int32_t *src, *dst; int64_t *bytes; double *w_xfer;       /* [n_edges] */
    int32_t *k0, *k1, *v0, *v1, *owner; uint8_t *cls;          /* [n_attrs] */
    int64_t *slow;                                            /* [2 n_slow] */
} hs_dot_host_t;

int hs_dot_parse(const uint8_t *text, int64_t len, hs_dot_info_t *info, void **handle,
                 void *stream);
int hs_dot_fetch(void *handle, const hs_dot_host_t *out, void *stream);
int hs_dot_csr_size(void *handle, int64_t *n, int64_t *m, void *stream);
int hs_dot_csr(void *handle, int64_t *out_ptr, int32_t *out_dst, int64_t *ids, double *w_cpu,
               double *w_gpu, double *w_xfer, int64_t *bytes, int32_t *root_host, void *stream);
int hs_dot_release(void *handle);
/* Python float(bytes) with the device's conversion, on the host (tests):
 * 0 ok, 1 ValueError, 2 undecided (exponent beyond +-100000) */
int hs_dot_py_float(const uint8_t *bytes, int64_t len, double *out);

#ifdef __cplusplus
}
#endif
#endif /* HETSCHED_B200_H */
