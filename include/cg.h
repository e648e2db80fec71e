/*
 * cg.h — C ABI of the B200-native computation-graph evaluator
 * (arXiv 1812.03770, "Owl's computation graph").
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * the CPU-program specification; section names in brackets.
 *
 * The library evaluates a computation graph G = (V, E, lambda, U)
 * [Def. 1, P:36-40] over fp32 ndarrays on one B200: it builds the graph node
 * by node [Operator layer, P:261-262], infers shapes eagerly [Shape, P:255-256],
 * optimises it (CSE, constant folding, dead-code elimination) [Optimiser,
 * P:264-280], plans one shared-block memory pool with Algorithm 1 applied to
 * fused kernel groups [Initialisation, P:292-364], and evaluates it with one
 * generated sm_100a kernel per fused elementwise/reduction group plus
 * hand-written kernels for dot/conv/pool/concat [Evaluation, P:366-367].
 * Update edges U are applied at the end of each evaluation [Graph, P:283].
 * Re-evaluation after cg_assign is incremental [P:25, P:42].
 *
 * Conventions
 *  - Element type: fp32 only.  Shapes are row-major; images NHWC, kernels HWIO.
 *  - State machine [static graph, P:249]:
 *      BUILD (cg_add_node / cg_add_update)
 *        -> cg_optimise (optional)
 *        -> cg_plan_memory (allocates, compiles; the graph is frozen)
 *        -> RUN (cg_assign / cg_eval / cg_read, repeatable).
 *    Calls out of order return CG_E_STATE.
 *  - Errors: functions return >= 0 on success and a negative cg_status on
 *    failure; cg_last_error() gives a message naming the node and the rule.
 *    Numerical problems are never errors: they surface as non-finite values.
 *  - Ownership: the library owns all device memory (pool, Var/Const buffers,
 *    workspace).  CONST data and cg_assign sources are COPIED; caller memory
 *    is never aliased.  Pointers returned by cg_eval are BORROWED and stay
 *    valid until the next cg_assign, cg_eval or cg_destroy on that graph.
 *  - Threading: one graph per host thread; no internal locking.  All device
 *    work is enqueued on the stream given to cg_create (NULL = legacy default).
 *  - Host-only mode: cg_create(device = -1, ...) builds, optimises and plans
 *    without touching a GPU (structure only: folded Const values are not
 *    computed, nothing is allocated, cg_eval returns CG_E_NO_DEVICE).  It
 *    exists so the host compiler's decisions can be tested on a CPU box; it
 *    performs no arithmetic on data and is not a fallback.
 */
#ifndef CG_H
#define CG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cg_graph cg_graph;  /* opaque; one per device per process thread */
typedef int32_t cg_node;           /* dense id >= 0 in creation order; never renumbered */

/* Operation variant type [Type layer, P:252-253].  Elementwise binary ops use
 * numpy trailing-dimension broadcasting. */
typedef enum cg_op {
  CG_VAR = 0,          /* arity 0: a variable input [Def. 1; Graph, P:283] */
  CG_CONST,            /* arity 0: constant data, copied at add time */
  CG_ADD, CG_SUB, CG_MUL, CG_DIV, CG_POW, CG_MAX2, CG_MIN2,   /* binary */
  CG_RELU_GRAD,        /* (z, g) -> z > 0 ? g : +0 */
  CG_FMA,              /* (a, b, c) -> a*b + c, one rounding [P:273] */
  CG_NEG, CG_ABS, CG_SQRT, CG_EXP, CG_LOG, CG_SIN, CG_COS, CG_TANH,
  CG_RELU,             /* x > 0 ? x : +0 */
  CG_SUM, CG_MAX,      /* reduce axes [a0, a1), keepdims (reduced extents become 1) */
  CG_DOT,              /* rank 2: C = op(A) op(B); attrs ta, tb */
  CG_CONV2D,           /* (x NHWC, w HWIO) -> y NHWC; attrs sh, sw, pad [Conv2d of padding * int array, P:253] */
  CG_CONV2D_BWD_INPUT, /* (dy, w) -> dx; attrs sh, sw, pad, h, w (input spatial size) */
  CG_CONV2D_BWD_KERNEL,/* (x, dy) -> dw HWIO; attrs sh, sw, pad, kh, kw */
  CG_MAXPOOL2D,        /* x -> window max; attrs kh, kw, sh, sw, pad (SAME pads with -inf) */
  CG_MAXPOOL2D_BWD,    /* (x, dy) -> dx: dy to the first maximal element of each window */
  CG_AVGPOOL2D,        /* mean over in-bounds window elements */
  CG_CONCAT,           /* n >= 1 inputs along attr axis */
  CG_RESHAPE,          /* row-major reinterpretation to attr dims (numel preserved) */
  CG_ALLREDUCE_SUM,    /* sum over data-parallel ranks (identity at world = 1) [P:26, P:42] */
  CG_FUSED_ADAGRAD,    /* (g, s, lr, eps) -> lr*g / (sqrt(s) + eps), computed in f64, one rounding;
                          produced by the AdaGrad rewrite (cg_set_rewrites) [Fused_Adagrad, P:273-277] */
  CG_NUM_OPS
} cg_op;

/* Operation parameters.  Fields not used by an op are ignored.
 * Padding convention (TF/Owl): pad = 0 VALID: out = floor((in - k)/s) + 1;
 * pad = 1 SAME: out = ceil(in/s), total padding max((out-1)s + k - in, 0),
 * floor half before. */
typedef struct cg_attr {
  int32_t ndim;            /* VAR/CONST: rank (0 = scalar); RESHAPE: target rank */
  int64_t dims[8];         /* VAR/CONST shape; RESHAPE target dims */
  const float* host_data;  /* CONST (required) / VAR (optional initial value):
                              numel fp32 values, row-major, host memory, copied */
  int32_t a0, a1;          /* SUM/MAX: axes [a0, a1), 0 <= a0 < a1 <= rank */
  int32_t ta, tb;          /* DOT: transpose A / B */
  int32_t sh, sw, pad;     /* conv/pool strides; pad 0 = VALID, 1 = SAME */
  int32_t kh, kw;          /* pool window; CONV2D_BWD_KERNEL kernel extent */
  int32_t h, w;            /* CONV2D_BWD_INPUT: spatial size of the forward input */
  int32_t axis;            /* CONCAT axis */
} cg_attr;

typedef enum cg_status {
  CG_OK = 0,
  CG_E_ARITY = -1,         /* wrong number of inputs / missing attribute */
  CG_E_BAD_NODE = -2,      /* unknown node id */
  CG_E_SHAPE = -3,         /* broadcast / dot / conv / reshape mismatch, at add time */
  CG_E_NOT_VAR = -4,       /* update or assign target is not a Var (Def. 1) */
  CG_E_DUP_UPDATE = -5,    /* a Var receives two update edges */
  CG_E_UPDATE_SHAPE = -6,  /* update source and target shapes differ */
  CG_E_NOT_PLANNED = -7,   /* cg_eval/cg_read on a node that is not a planned root */
  CG_E_SIZE = -8,          /* cg_assign/cg_read byte count != numel * 4 */
  CG_E_STATE = -9,         /* call out of the BUILD -> OPTIMISED -> PLANNED order */
  CG_E_CUDA = -10, CG_E_NCCL = -11, CG_E_NVRTC = -12, CG_E_OOM = -13,
  CG_E_ARG = -14,          /* NULL pointer / bad flag / bad rank */
  CG_E_NO_DEVICE = -15     /* evaluation requested on a host-only graph */
} cg_status;

/* Data-parallel placement [P:26]: rank r of `world` processes; the 128-byte
 * NCCL unique id comes from cg_nccl_unique_id on rank 0, broadcast by the
 * caller.  NULL or world == 1: single GPU, ALLREDUCE_SUM is the identity.
 * nccl_unique_id == NULL with world > 1: no NCCL communicator; the graph must be
 * planned with CG_PLAN_FUSED_COLL (peer-memory collectives). */
typedef struct cg_dist {
  int32_t rank, world;
  const void* nccl_unique_id;
} cg_dist;

/* Structural effect of cg_optimise; equal to the oracle's counts. */
typedef struct cg_report {
  int32_t cse_merged, cf_folded, dce_removed;
  /* pattern rewrites requested with cg_set_rewrites (0 otherwise) [P:273-279] */
  int32_t rw_identity;   /* x+0, 0+x, x-0, x*1, 1*x, x/1 -> x */
  int32_t rw_zeroed;     /* x*0, 0*x -> Const zeros */
  int32_t rw_fma;        /* ADD(MUL(a,b), c) -> FMA(a,b,c) */
  int32_t rw_adagrad;    /* DIV(MUL(lr,g), ADD(SQRT(s),eps)) -> FUSED_ADAGRAD(g,s,lr,eps) */
} cg_report;

/* Memory plan summary [P:292-364]. */
typedef struct cg_plan_info {
  int32_t n_groups;          /* kernel groups in evaluation order Gamma */
  int32_t n_blocks;          /* shared pool blocks */
  int32_t n_kernels;         /* distinct generated kernels compiled */
  int32_t n_fused;           /* groups computed inside another group's kernel (f2: DOT / CONV / pool epilogues, pool prologues; sibling 1x1 convs merged into one GEMM) */
  uint64_t pool_bytes;       /* sum of align256(block bytes) */
  uint64_t plan_bytes;       /* sum of exact block bytes */
  uint64_t external_bytes;   /* Var + Const buffers */
  uint64_t workspace_bytes;  /* kernel scratch outside Algorithm 1 (reduction partials) */
  uint64_t unshared_bytes;   /* eager baseline: one fresh buffer per raw-graph op node */
} cg_plan_info;

enum { CG_PLAN_INCREMENTAL = 1u, /* pin Var frontiers, fresh blocks for kept values,
                                    signature-pure groups: minimal recompute sets */
       CG_PLAN_NO_FUSION = 2u,   /* one kernel per node (node-level Algorithm 1) */
       CG_PLAN_FUSED_COLL = 4u   /* ALLREDUCE_SUM (+ its elementwise update) as one
                                    peer-memory kernel instead of NCCL (f3; same plan) */ };
enum { CG_EVAL_NO_UPDATE = 1u,   /* skip update_iopair at the end of this evaluation */
       CG_EVAL_FULL = 2u,        /* ignore validity: recompute every group */
       CG_EVAL_SYNC = 4u         /* block the host until the evaluation finished */ };
enum { CG_DUMP_GRAPH = 0, CG_DUMP_PLAN = 1 };
enum { CG_RW_IDENTITY = 1u, CG_RW_FMA = 2u, CG_RW_ADAGRAD = 4u, CG_RW_ALL = 7u };

/* Create a graph on CUDA `device` (-1: host-only planning mode).  `cuda_stream`
 * is a cudaStream_t (NULL: default stream).  Returns NULL on failure
 * (cg_last_error(NULL) explains). */
cg_graph* cg_create(int device, void* cuda_stream, const cg_dist* dist);

/* Add a vertex [Operator layer; add_node S:51-59].  `inputs` are
 * existing node ids (duplicates allowed: x <- y*y).  The output shape is
 * inferred immediately [P:255-256].  Returns the new id (>= 0) or a cg_status. */
cg_node cg_add_node(cg_graph* g, cg_op op, const cg_node* inputs, int32_t n_inputs,
                    const cg_attr* attr);

/* Add the update edge (u, var) in U [Def. 1; iopair P:283]: at the end
 * of every evaluation var <- copy(value(u)) with parallel-assignment semantics.
 * var must be a Var with u's shape; at most one edge per Var. */
int cg_add_update(cg_graph* g, cg_node u, cg_node var);

/* Request the paper's pattern rewrites [Optimiser, P:273-279] for the next
 * cg_optimise (BUILD state only): CG_RW_IDENTITY removes "useless calculations"
 * (adding zero, dividing by one, multiplying by zero or one), CG_RW_FMA fuses a
 * single-consumer MUL into its ADD, CG_RW_ADAGRAD fuses the AdaGrad
 * adjusted-gradient subgraph.  They run to a fixpoint before CSE/CF/DCE; kept
 * values (outputs, update sources) are never removed or absorbed.  Default: none. */
int cg_set_rewrites(cg_graph* g, uint32_t flags);

/* Declare the graph's outputs [a graph is "defined by its inputs and outputs
 * nodes", P:283] and run CSE -> constant folding -> DCE [P:264-272].  Folded
 * values are computed once, on the device, by the same kernels as evaluation.
 * `report` may be NULL.  Node ids stay valid: merged ids resolve to their
 * representative everywhere. */
int cg_optimise(cg_graph* g, const cg_node* outputs, int32_t n_outputs, cg_report* report);

/* Order (post-order DFS from the outputs, then the update sources [P:312]),
 * fuse, plan the pool with Algorithm 1 [P:323-362], allocate, and compile the
 * group kernels for sm_100a.  `outputs` must be live nodes.  `info` may be NULL. */
int cg_plan_memory(cg_graph* g, const cg_node* outputs, int32_t n_outputs, uint32_t flags,
                   cg_plan_info* info);

/* Copy `nbytes` (== numel*4) from `src` (device memory if src_on_device,
 * else host memory) into Var `var`; its descendants become dirty [P:42].
 * Asynchronous on the graph's stream; the source must stay valid until then. */
int cg_assign(cg_graph* g, cg_node var, const void* src, size_t nbytes, int src_on_device);

/* Evaluate [P:366-367]: recompute exactly the groups needed for `outputs`
 * (planned roots) that are not valid [P:25], then apply the update edges
 * [P:283] unless CG_EVAL_NO_UPDATE.  On success out_dev_ptrs[i] (if not NULL)
 * receives a borrowed device pointer to outputs[i]'s fp32 value. */
int cg_eval(cg_graph* g, const cg_node* outputs, int32_t n_outputs,
            const float** out_dev_ptrs, uint32_t flags);

/* Copy the current value of a planned root, Var or Const to host memory
 * (nbytes == numel*4); synchronises the graph's stream. */
int cg_read(cg_graph* g, cg_node node, void* host_dst, size_t nbytes);

void cg_destroy(cg_graph* g);

/* Message of the last failing call on g (or of cg_create when g is NULL). */
const char* cg_last_error(const cg_graph* g);

/* Fused AllReduce + update over peer memory [P:26 "natural support for parallel
 * and distributed computing"; SURVEY §8(f) f3].  With CG_PLAN_FUSED_COLL every
 * ALLREDUCE_SUM group is one kernel that sums the gradient over all ranks in rank
 * order 0..P-1 -- reading the other ranks' pools through CUDA IPC mappings (NVLink)
 * at the same pool offset (every rank plans the same graph) -- and applies the
 * elementwise update chain that consumes it (e.g. W - lr * g, Var / Const operands)
 * before storing; independent collectives of one executor step are one launch.  A
 * system-scope flag barrier orders the reads after every rank's gradient is final
 * and keeps gradients alive until every rank has read them.
 *   cg_coll_handle: after cg_plan_memory, writes this rank's 128-byte handle
 *     (cudaIpcMemHandle of the pool, then of the flag words); returns 128.
 *   cg_coll_connect: `handles` = world x 128 bytes in rank order (gathered by the
 *     caller, e.g. over torch.distributed); maps the peers.  Required before the
 *     first cg_eval when world > 1 (CG_E_STATE otherwise); not needed at world 1.
 * Errors: CG_E_STATE (graph not planned with the flag), CG_E_SIZE (cap < 128),
 * CG_E_ARG (world differs from cg_create's), CG_E_CUDA (IPC failure). */
int cg_coll_handle(cg_graph* g, void* out, size_t cap);
int cg_coll_connect(cg_graph* g, const void* handles, int32_t world);

/* 128-byte NCCL unique id for cg_dist (call on rank 0 only). */
int cg_nccl_unique_id(void* out128);

/* ---- introspection (tests) ---- */
/* Canonical JSON of the optimised graph (CG_DUMP_GRAPH) or the plan
 * (CG_DUMP_PLAN): sorted keys, no whitespace, integers and op names only.
 * Writes at most cap bytes incl. NUL; returns the full length (excl. NUL). */
int64_t cg_dump_json(cg_graph* g, int what, char* buf, size_t cap);
/* How many times node's group has been launched (incremental invariant). */
int64_t cg_eval_count(const cg_graph* g, cg_node node);
/* Shape of a node: writes up to 8 dims, returns the rank (or a cg_status). */
int32_t cg_node_shape(const cg_graph* g, cg_node node, int64_t* dims8);
/* Number of device kernel launches enqueued by this graph so far. */
int64_t cg_launch_count(const cg_graph* g);
/* Executor order with batched collectives (the paper's "natural
 * support for parallel and distributed computing"), on synthetic access
 * sets: ng groups in Gamma order, active[g] (NULL: all), the pool blocks group g
 * reads rd_idx[rd_ptr[g]:rd_ptr[g+1]] and writes wr_idx[wr_ptr[g]:wr_ptr[g+1]],
 * uses_ws[g] (kernel workspace), is_coll[g] (ALLREDUCE_SUM).  Writes the issue
 * order to order[] and a step id per entry to step[] (entries with one step id
 * are collectives issued in one ncclGroupStart/End); returns the number of
 * scheduled groups or a cg_status.  Host only; caller owns every buffer
 * (order, step: ng entries).  The executor uses the same routine. */
int32_t cgx_collective_schedule(int32_t ng, const uint8_t* active, const int32_t* rd_ptr,
                                const int32_t* rd_idx, const int32_t* wr_ptr, const int32_t* wr_idx,
                                const uint8_t* uses_ws, const uint8_t* is_coll, int32_t* order,
                                int32_t* step);
/* Collective batches (ncclGroupStart/End pairs) g has issued, captured ones included. */
int64_t cgx_coll_batches(const cg_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* CG_H */
