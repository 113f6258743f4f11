/*
 * kr_engine.h — C ABI of the B200 gradient oracle (libkrcuda.so).
 *
 * Drop-in replacement for the reference's gradient boundary
 *   class GradientEngine { Vec Ax(x2); Vec ATx(x1); int64 flops(); }
 *   (/root/reference/proj/include/kronriver/solver.hpp:21-27)
 * implemented there by FactoredEngine (solver.hpp:30-40) over
 *   matvec          (engine.hpp:58-93)   y = (Ahat + U M^-1 V^T) x
 *   matvecTranspose (engine.hpp:96-133)  x = (Ahat + U M^-1 V^T)^T y
 * and of the solver step that drives it, dcfrSolve (solver.hpp:343-404)
 * with bestResponseValue / exploitability (solver.hpp:292-331).
 *
 * Plain pointers and sizes only; no exceptions cross the ABI.  Status codes
 * mirror the reference's error taxonomy (errors.hpp:11-58).  There is no CPU
 * fallback: creating an engine without a CUDA device fails with KR_NO_DEVICE.
 */
#ifndef KR_ENGINE_H
#define KR_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* errors.hpp:22-58 codes, plus two device-side codes. */
enum kr_status {
  KR_OK = 0,
  KR_INVALID_INPUT = 1,      /* InvalidInputError  "INVALID_INPUT"      */
  KR_PARSE = 2,              /* ParseError         "PARSE"              */
  KR_IO = 3,                 /* IoError            "IO"                 */
  KR_GUARD_EXCEEDED = 4,     /* GuardError         "GUARD_EXCEEDED"     */
  KR_DEGENERATE_BELIEFS = 5, /* DegenerateBeliefsError                  */
  KR_CONTRACT = 6,           /* ContractError      "CONTRACT"           */
  KR_CUDA = 7,               /* CUDA runtime failure                    */
  KR_NO_DEVICE = 8           /* no CUDA device: no CPU fallback exists  */
};

typedef struct kr_engine kr_engine;
typedef struct kr_solver kr_solver;

/* One compressed factor in the reference's storage order
 * (Eigen::SparseMatrix compressed arrays, linalg.hpp:12-16):
 * outer[outer_size+1], inner[nnz], val[nnz]; inner indices ascending. */
typedef struct {
  int64_t outer_size;
  const int64_t* outer;
  const int32_t* inner;
  const double* val;
} kr_compressed;

/* Sparsification (sparsify.hpp:110-121): A = Ahat + U M^-1 V^T. */
typedef struct {
  int64_t rows, cols, k;
  kr_compressed ahat; /* CSR rows x cols   */
  kr_compressed u;    /* CSR rows x k      */
  kr_compressed m;    /* CSC k x k, unit lower triangular */
  kr_compressed v;    /* CSC cols x k      */
  /* Optional layout hint: sequences per hand of the row / column player
   * (KronPayoff::flat, kron.hpp:124-126).  0 = unknown. */
  int32_t n1, n2;
} kr_factors;

/* Engine flags.  Host-buffer calls (kr_engine_ax / kr_engine_atx) on a
 * multi-board engine pipeline over up to four board groups, overlapping the
 * host<->device copies of one group with the kernels of another;
 * KR_FLAG_SINGLE_PART disables that (one copy, kernels, one copy; the
 * environment variable KR_GROUPS=<n> sets the group count). */
#define KR_FLAG_DEFAULT 0u
#define KR_FLAG_SINGLE_PART 1u

/* One river board in Kronecker form (kron.hpp:104-132): the payoff block of
 * hand pair (i, j) is pi_ij (F + W_ij S) with pi_ij = lambda1_i lambda2_j
 * [hands disjoint] and W_ij = sign(key1_i - key2_j).  Hands of each player are
 * strength-sorted ascending (kron.hpp:74-83); cards are ids 0..51. */
typedef struct {
  int32_t m1, m2, n1, n2;
  const uint32_t* key1;   /* [m1] packed strength keys (cards.hpp:167-194) */
  const uint32_t* key2;   /* [m2] */
  const uint8_t* cards1;  /* [2*m1] */
  const uint8_t* cards2;  /* [2*m2] */
  const double* lambda1;  /* [m1] mu1 / sqrt(beta) (kron.hpp:163)  */
  const double* lambda2;  /* [m2] */
  kr_compressed F;        /* CSR n1 x n2 fold payments (skeleton.hpp:332-349) */
  kr_compressed S;        /* CSR n1 x n2 showdown stakes */
} kr_kron_board;

/* Implicit Kronecker engine (the "showdown/fold factors as segmented prefix
 * scans with card-removal corrections" of the north star; SURVEY.md 8(f)
 * row 1).  Same products as kr_engine_ax / kr_engine_atx with nothing
 * materialised: per board it streams x and y (~0.8 MB) instead of the
 * factors (~76 MB).  Results equal referenceMatvec(T) (kron.hpp:211-254) up
 * to rounding (summation order differs); flops() counts its multiply-adds. */
int kr_engine_create_kron(const kr_kron_board* boards, int nboards, int device, uint32_t flags, kr_engine** out);

/* Technique B with postprocessing (sparsify.hpp:246-406) built ON THE DEVICE
 * from one board's KronPayoff pieces, bit-exact against
 * the host builder, downloaded into host arrays in the reference's storage
 * order (view: valid while f lives; usable with kr_engine_create).  seconds:
 * device time of the build (CUDA events, downloads included). */
typedef struct kr_devfactors kr_devfactors;
int kr_factors_build_device(const kr_kron_board* b, int device, kr_devfactors** out);
int kr_devfactors_view(const kr_devfactors* f, kr_factors* out);
double kr_devfactors_seconds(const kr_devfactors* f);
void kr_devfactors_free(kr_devfactors* f);

/* The factored engine (Technique B with postprocessing) built entirely on the
 * device from the boards' KronPayoff pieces: factors generated row by row into
 * the engine's layout, no factor arrays and no layout work on the host
 * (SURVEY.md 8(f) row 3).  Products are bitwise those of kr_engine_create on
 * the host builder's factors. */
int kr_engine_create_device_b(const kr_kron_board* boards, int nboards, int device, uint32_t flags,
                              kr_engine** out);

/* The Kronecker-factored engine: Technique B with postprocessing
 * (sparsify.hpp:246-406) kept as its hand-space factors (lambda1, lambda2, the
 * blocked-hand lists of Hx, the sparsity of Y = D W) and the tree's F and S,
 * with every Kronecker product expanded on the fly (a few hundred KB per board
 * instead of the ~150 MB of expanded factors).  Products are BITWISE those of
 * kr_engine_create on the host builder's Technique B post factors (same terms,
 * same order, engine.hpp:58-133); one fused launch per product, one CTA per
 * (sequence, board).  Boards of at most 2047 hands per side.  Replaces
 * FactoredEngine(techniqueB + postprocess) (solver.hpp:30-40). */
int kr_engine_create_kfactored(const kr_kron_board* boards, int nboards, int device, uint32_t flags,
                               kr_engine** out);

/* Create an engine for one Sparsification on CUDA device `device`.
 * Replaces FactoredEngine(const Sparsification&) (solver.hpp:32); the
 * factors are copied to HBM, so the caller may free them afterwards. */
int kr_engine_create(const kr_factors* f, int device, uint32_t flags, kr_engine** out);

/* Block-diagonal engine over `nboards` independent Sparsifications (the
 * chance/board dimension of a turn endgame):
 * x and y are the per-board vectors concatenated in board order. */
int kr_engine_create_boards(const kr_factors* boards, int nboards, int device, uint32_t flags,
                            kr_engine** out);

int kr_engine_destroy(kr_engine* e);

/* rows, cols, k, nnz(ahat), nnz(u), nnz(m), nnz(v), identity(M) */
int kr_engine_dims(const kr_engine* e, int64_t out[8]);

/* GradientEngine::Ax (solver.hpp:24, engine.hpp:58): y[rows] = A x[cols].
 * HOST buffers (pinned buffers from kr_host_alloc transfer fastest).
 * KR_INVALID_INPUT on a size mismatch (engine.hpp:59-61), KR_CONTRACT when M
 * is not unit lower triangular (engine.hpp:35-36). */
int kr_engine_ax(kr_engine* e, const double* x, int64_t nx, double* y, int64_t ny);

/* GradientEngine::ATx (solver.hpp:25, engine.hpp:96): x[cols] = A^T y[rows]. */
int kr_engine_atx(kr_engine* e, const double* y, int64_t ny, double* x, int64_t nx);

/* Both products of one pair on HOST buffers: ax[rows] = A x[cols] and
 * atx[cols] = A^T y[rows], the two directions' copies on the bus at once
 * (host->device of x and y, device->host of both results, pipelined over
 * board groups) and their kernels side by side; returns when both results
 * are in host memory.  Results are bitwise those of kr_engine_ax then
 * kr_engine_atx.  Pinned buffers (kr_host_alloc) replay a captured graph from
 * the second call with the same pointers on.  No reference counterpart: the
 * reference calls Ax and ATx one after the other (solver.hpp:21-27,
 * bestResponseValue's two calls at a checkpoint are independent, 299). */
int kr_engine_pair(kr_engine* e, const double* x, int64_t nx, double* ax, int64_t nax, const double* y, int64_t ny,
                   double* atx, int64_t natx);

/* A queue of `count` independent pairs on HOST buffers: axs[i] = A xs[i] and
 * atxs[i] = A^T ys[i] for i < count (arrays of buffer pointers; the same
 * buffer may appear in several entries).  Each result is bitwise that of
 * kr_engine_pair on the same pair.  The input copies of pair i + 1 and the
 * output copies of pair i - 1 overlap pair i's kernels (two device slots per
 * direction), so with pinned buffers the bus runs inputs and outputs at once,
 * back to back.  Inputs are read at unspecified times during the call: no
 * output buffer may alias any input buffer of the queue.  Returns when every
 * result is in host memory.  The reference's counterpart is its benchmark
 * loop of independent products (tools/main.cpp:313-323). */
int kr_engine_pair_queue(kr_engine* e, int64_t count, const double* const* xs, int64_t nx, double* const* axs,
                         int64_t nax, const double* const* ys, int64_t ny, double* const* atxs, int64_t natx);

/* Device-pointer variants, enqueued on `stream` (NULL = the engine's own
 * stream); asynchronous with respect to the host. */
int kr_engine_ax_device(kr_engine* e, const double* x_dev, double* y_dev, void* stream);
int kr_engine_atx_device(kr_engine* e, const double* y_dev, double* x_dev, void* stream);

/* Both products of one pair, ax_dev = A x_dev and atx_dev = A^T y_dev, in
 * flight together: A^T y runs on an engine-owned side stream forked from
 * `stream` and joined back into it, so the latency-bound stages of each
 * direction (transposes, M solves, short SpMVs) overlap the other direction's
 * bandwidth-bound SpMV; above ~8 GB of factors per pair (KR_PAIR_SERIAL_GB),
 * where each direction is bandwidth-bound alone, the two run one after the
 * other on `stream`.  Results are bitwise those of kr_engine_ax_device /
 * kr_engine_atx_device (each direction has its own scratch).  x_dev must not
 * alias atx_dev, nor y_dev ax_dev.  No reference counterpart: the reference
 * calls Ax and ATx one after the other (GradientEngine, solver.hpp:21-27). */
int kr_engine_pair_device(kr_engine* e, const double* x_dev, double* ax_dev, const double* y_dev, double* atx_dev,
                          void* stream);

/* GradientEngine::flops() (solver.hpp:26, 35): cumulative multiply-adds,
 * counted with the reference rule nnz(V)+nnz(U)+nnz(Ahat)+[M!=I](nnz(M)-k)
 * per product (engine.hpp:72,77,90-91,110-131). */
int64_t kr_engine_flops(const kr_engine* e);
/* multiply-adds of the last product (GradientWorkspace::flops) */
int64_t kr_engine_last_flops(const kr_engine* e);

/* The engine's CUDA stream (cudaStream_t) and device. */
void* kr_engine_stream(const kr_engine* e);
int kr_engine_device(const kr_engine* e);

/* Kernel launches issued by this engine since creation (both directions). */
int64_t kr_engine_launches(const kr_engine* e);

/* SelfCheck mode, the device counterpart of SelfCheckEngine
 * (solver.hpp:67-99): every `every`-th product of e (calls 0, every,
 * 2 every, ..., counted over kr_engine_ax / _atx / _pair and the device
 * variants) is replayed through `reference` (typically the implicit engine
 * over the same boards: the block formula, kron.hpp:211-254) and compared on
 * the device; max|got - exp| > tol (1 + max|exp|) makes the next host-buffer
 * call, kr_solver_run on e, or kr_engine_selfcheck_status return
 * KR_CONTRACT (the reference throws ContractError).  Solvers on a
 * self-checked engine run iteration by iteration (no graph replay), so every
 * product is checked on schedule.  reference = NULL turns it off.  The
 * reference defaults are every = 500, tol = 1e-8. */
int kr_engine_set_selfcheck(kr_engine* e, kr_engine* reference, int every, double tol);
/* Checks made so far, the worst err / (tol (1 + max|exp|)) seen; KR_CONTRACT
 * if a check has failed. */
int kr_engine_selfcheck_status(kr_engine* e, int64_t* checks, double* worst);

/* Pinned host memory for the host-buffer entry points. */
void* kr_host_alloc(int64_t bytes);
void kr_host_free(void* p);

/* Last error message of the calling thread, and its status code. */
const char* kr_last_error(int* code);

/* Number of CUDA devices visible (0 on a machine without a GPU). */
int kr_device_count(void);

/* The bounds-checked build (KR_CHECKED; lib/libkrcuda_checked.so): the number
 * of device allocations whose guard zones were found overwritten (live ones
 * now, freed ones when they were freed), 0 when all are intact; -1 in the
 * normal build.  Synchronises the device.  No reference counterpart (the
 * reference's sanitizer builds). */
int64_t kr_checked_verify(void);

/* The checked build's own test (-1 in the normal build): mode 0 writes one
 * double past a 100-double allocation and returns the number of corrupted
 * guard zones found (1); mode 1 does it behind a failing device index check,
 * which traps (returns minus the CUDA error; the context is lost). */
int64_t kr_checked_selftest(int mode);

/* ---------------------------------------------------------------------------
 * Solver step on the device: DCFR with alternating updates
 * (solver.hpp:343-404), regret matching (166-194), sequence form (197-218),
 * regret sweep (222-260), discounting (262-264), averaging (381-387), and
 * best response / exploitability at checkpoints (292-331).
 * ------------------------------------------------------------------------- */

/* Treeplex of one player (skeleton.hpp:89-126): that player's decision nodes
 * in preorder.  node i has parent sequence node_parent_seq[i] (0 = empty
 * sequence) and actions action_seq[node_action_ptr[i] .. node_action_ptr[i+1])
 * (1-based sequence ids, skeleton.hpp:84). */
typedef struct {
  int32_t n_seq;
  int32_t n_nodes;
  const int32_t* node_parent_seq;
  const int32_t* node_action_ptr;
  const int32_t* action_seq;
} kr_treeplex;

/* DcfrParams (solver.hpp:101-109), plus the update rule (not in the
 * reference, whose only solver is DCFR):
 *   KR_RULE_DCFR  the reference's dcfrSolve (solver.hpp:343-404);
 *   KR_RULE_CFRP  each player's regrets discounted right after its sweep and
 *                 its strategy regret-matched on them; with alpha = +inf and
 *                 beta = -inf that is CFR+ (R <- max(R + r, 0)), gamma = 1
 *                 gives its linear averaging;
 *   KR_RULE_PRMP  predictive regret matching+: as CFRP, strategy matched on
 *                 R + r (the last instantaneous regret as the prediction).
 * alpha / beta = +-inf use the limits 1 / 0 of t^e / (t^e + 1). */
#define KR_RULE_DCFR 0
#define KR_RULE_CFRP 1
#define KR_RULE_PRMP 2
typedef struct {
  double alpha, beta, gamma;
  int32_t max_iters;
  double target_exploitability;
  int32_t checkpoint_every;
  int32_t rule; /* KR_RULE_* (0 = the reference's DCFR) */
} kr_dcfr_params;

/* Caller-owned result buffers (DcfrResult, solver.hpp:133-140).  trace_* hold
 * up to trace_cap checkpoints; per-board arrays hold trace_cap*nboards values
 * (checkpoint-major) when non-NULL.  avg1/avg2 receive the final average
 * sequence-form strategies when non-NULL. */
typedef struct {
  int32_t iterations;
  double exploitability;
  int64_t gradient_flops;
  int32_t trace_len;
  int32_t trace_cap;
  int32_t* trace_iter;
  double* trace_expl;
  double* trace_br1;        /* summed over boards */
  double* trace_br2;
  double* trace_board_br1;  /* [trace_cap * nboards] or NULL */
  double* trace_board_br2;
  double* avg1;             /* [rows] or NULL */
  double* avg2;             /* [cols] or NULL */
  double seconds;           /* device time of the whole solve (CUDA events) */
} kr_dcfr_result;

/* Bind a solver to an engine.  hands1[b], hands2[b]: hand counts of board b
 * (rows = sum hands1[b] * p1->n_seq, cols = sum hands2[b] * p2->n_seq);
 * pot = 2 * potContribution (solver.hpp:329).  The engine must outlive the
 * solver. */
int kr_solver_create(kr_engine* e, const kr_treeplex* p1, const kr_treeplex* p2, int nboards,
                     const int32_t* hands1, const int32_t* hands2, double pot, kr_solver** out);
int kr_solver_destroy(kr_solver* s);

/* dcfrSolve.  exploitability = sum_b (br1_b + br2_b) / 2 / pot / nboards
 * (the chance root picks a board uniformly; nboards = 1 is the reference). */
int kr_solver_run(kr_solver* s, const kr_dcfr_params* p, kr_dcfr_result* r);

/* bestResponseValue (solver.hpp:292-321) against a HOST opponent strategy;
 * value summed over boards (per-board values in board_values if non-NULL).
 * KR_INVALID_INPUT on a malformed strategy (validateSequenceStrategy,
 * solver.hpp:266-286). */
int kr_solver_best_response(kr_solver* s, int player, const double* opp, int64_t n, double* value,
                            double* board_values);

/* Kernel launches issued by the solver (its own kernels, not the engine's). */
int64_t kr_solver_launches(const kr_solver* s);

/* Incremental form of kr_solver_run, for drivers that combine boards held by
 * several ranks between checkpoints (one allreduce of the gap scalars per
 * checkpoint).  begin: zero regrets/averages and form the
 * uniform strategies (solver.hpp:348-364); iterate: n DCFR iterations
 * (365-388); checkpoint: best-response values of the current average profile
 * per board (389-392, 325-331); averages: the normalised average strategies
 * (400-401). */
int kr_solver_begin(kr_solver* s, double alpha, double beta, double gamma);
/* Update rule (KR_RULE_*) of the following begin / iterate calls; rules other
 * than DCFR need a treeplex whose parent sequences belong to earlier nodes
 * (every reference skeleton), else KR_INVALID_INPUT. */
int kr_solver_set_rule(kr_solver* s, int rule);
/* Which kernel runs `player`'s DCFR step (0 or 1): 2 = compiled for the
 * player's treeplex at solver creation (NVRTC, kr_jit.cu: one thread per
 * hand, regrets in registers), 1 = the generic team kernel, 0 = the generic
 * one-thread-per-hand kernel; -1 for a bad argument.  `why` (optional)
 * receives the reason the compiled step is not used (empty when it is).
 * All three give bitwise-identical results. */
int kr_solver_step_kind(const kr_solver* s, int player, const char** why);
/* The CUDA C the compiled step is generated from, for treeplex t and update
 * rule (KR_RULE_*): copies up to cap bytes (NUL-terminated) into buf when buf
 * is non-NULL and returns the source length, or -1 when the treeplex is not
 * level-ordered (or, with KR_JIT_SOURCE_GROUPS=g, does not split into g warp
 * groups: the single-board form).  Needs no device (inspection and compile
 * tests). */
int64_t kr_jit_step_source(const kr_treeplex* t, int rule, char* buf, int64_t cap);
int kr_solver_iterate(kr_solver* s, int n);
int kr_solver_checkpoint(kr_solver* s, double* board_br1, double* board_br2);
int kr_solver_averages(kr_solver* s, double* avg1, double* avg2);
int kr_solver_iteration(const kr_solver* s);

/* Turn endgames (a betting round above the river boards; beyond the
 * reference).  The payoff is block diagonal: turnEng covers the
 * turn block (m hands x the turn trees' sequences); riverEngs[t] covers
 * continuation t's river block over all boards (board-major, each board's hand
 * order).  mb[b] = river hands of board b; riverToTurn[r] = the turn hand of
 * river hand r (board-major); sigma[2t + p] = player p's turn sequence leading
 * to continuation t; riverTrees[2t + p] its river treeplex; pot = 2 x the
 * turn contribution.  run: DCFR, CFR+ or PRM+ (kr_dcfr_params.rule) with the turn treeplex
 * composed as in DESIGN.md §4.8; avg1 / avg2 receive the full average
 * strategies (turn block, then each continuation's river block). */
typedef struct kr_turn_solver kr_turn_solver;
int kr_turn_solver_create(kr_engine* turnEng, int T, kr_engine* const* riverEngs, const kr_treeplex* turnTrees,
                          const kr_treeplex* riverTrees, int m, int nb, const int32_t* mb, const int32_t* riverToTurn,
                          const int32_t* sigma, double pot, kr_turn_solver** out);
int kr_turn_solver_run(kr_turn_solver* s, const kr_dcfr_params* p, kr_dcfr_result* r);
int kr_turn_solver_destroy(kr_turn_solver* s);
int64_t kr_turn_solver_launches(const kr_turn_solver* s);
/* Board sharding over ranks with a host-driven transport (e.g. a gloo
 * process group): each rank's solver holds the turn block and its own
 * boards.  fn(user) is called (stream synchronised) after the river steps of
 * every half-iteration and of every best response and must all-gather the
 * device buffer send (sizes[2] * max(boards_per_rank) doubles: this rank's
 * per-board river values) into the device buffer recv (world times that,
 * rank-major); both buffers stay the caller's.  The library then folds the
 * values in global board order, exactly as on one GPU, so the solve is
 * bitwise the one-GPU solve.  fn = NULL restores the single-rank solver. */
int kr_turn_solver_set_exchange(kr_turn_solver* s, void (*fn)(void*), void* user, int world, int rank,
                                const int32_t* boards_per_rank, double* send, double* recv);
/* rows of player 1's vector, of player 2's, exchanged values per board, river hands */
int kr_turn_solver_sizes(const kr_turn_solver* s, int64_t out[4]);

/* ---------------------------------------------------------------------------
 * Multi-GPU: one rank per GPU, boards sharded contiguously over the ranks
 * (rank r holds boards [sum boards_per_rank[<r], +boards_per_rank[r])).  The
 * turn payoff is block diagonal over boards, so products
 * need no communication; what crosses ranks is all-gathered and folded in
 * global board order on every rank, the fold of the one-GPU solver, so all
 * results are bitwise independent of the rank count.
 * Transport: NCCL over NVLink / NVSwitch, enqueued on the solver stream and
 * captured into its iteration graphs.
 * ------------------------------------------------------------------------- */
#define KR_COMM_ID_BYTES 128
typedef struct kr_comm kr_comm;
/* A fresh NCCL unique id (rank 0 creates it and shares it with the others). */
int kr_comm_unique_id(uint8_t* id);
/* One rank of an nranks communicator on CUDA device `device` (one process per
 * GPU): every rank calls it with the same id. */
int kr_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, kr_comm** out);
/* ndev ranks in one process, rank r on devices[r]: out[0..ndev). */
int kr_comm_init_all(int ndev, const int* devices, kr_comm** out);
int kr_comm_destroy(kr_comm* c);
int kr_comm_rank(const kr_comm* c);
int kr_comm_size(const kr_comm* c);

/* The solver's boards are this rank's shard of boards_per_rank (one entry per
 * rank of c).  From now on kr_solver_run / kr_solver_checkpoint report every
 * board of every rank in global order (result arrays sized for the total),
 * the exploitability averages over all boards, and checkpoint values travel
 * by an in-stream all-gather captured into the iteration graphs.  c = NULL
 * restores the single-rank solver. */
int kr_solver_set_comm(kr_solver* s, kr_comm* c, const int32_t* boards_per_rank);

/* Per-iteration exchange of the turn solver (its river values per turn hand,
 * board by board) over c: all-gathered in-stream, folded in global board
 * order (graphs stay on). */
int kr_turn_solver_set_comm(kr_turn_solver* s, kr_comm* c, const int32_t* boards_per_rank);

/* Per-kernel CUDA-event timing of the engine's SpMV launches (off by
 * default).  When enabled every SpMV launch is bracketed by events on the
 * engine's stream; kr_engine_kernel_times returns, for the four matrices
 * [V^T, U|Ahat, U^T, Ahat^T|V], the number of launches, their summed
 * milliseconds and the algorithmic bytes of one launch. */
int kr_engine_set_timing(kr_engine* e, int enabled);
/* Which of the four matrices the timing brackets (bit w = matrix w in the
 * order above; default 0xF).  Timing only the dominant kernel keeps the
 * events' own cost (~1.5% of a pair for all four) out of a timed region. */
int kr_engine_set_timing_mask(kr_engine* e, int mask);
int kr_engine_kernel_times(kr_engine* e, int64_t launches[4], double ms[4], double bytes[4]);

#ifdef __cplusplus
}
#endif

#endif /* KR_ENGINE_H */
