/*
 * sel.h — C ABI of libsel: the exact-selectivity probe on B200 (sm_100a).
 *
 * The method (Shin 2018, "Novel Selectivity Estimation Strategy for Modern DBMS",
 * arXiv 1806.08384; PAPER.md = /root/reference/PAPER.md):
 *   - sel_count    = Listing 3.1: `SELECT COUNT(*) FROM R WHERE <pushed-down
 *                    predicate>`, "the exact cardinality of the given selection",
 *                    computed by iterating "through all the tuples and simply increase a counter
 *                    whenever it finds a tuple which satisfies the given condition".
 *   - sel_pushdown = materialising sigma(R) with the projection pushed down (PAPER.md:141, 235,
 *                    329; Algorithm 1 lines 380-383 / Execute): selected row ids
 *                    plus projected columns, with the Execute(isSPD, maxSize) capacity gate
 *                    "if count > maxSize throw" as a distinguishable outcome.
 *
 * Everything the library touches on the device is caller-owned (torch tensors in the Python
 * binding). The library never allocates, frees or copies column data; it owns only metadata and
 * a small per-context scratch area (tile status words, per-CTA partials, a pinned 16-byte result
 * slot). A context is not re-entrant: one call at a time per context.
 *
 * Errors: calls returning sel_status return the code; calls returning uint64_t return SEL_ERR on
 * a hard error. Both set a thread-local status + message readable with sel_last_error() and
 * sel_last_error_message(). A successful call sets the thread-local status to SEL_OK.
 */
#ifndef SEL_H_
#define SEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEL_ABI_VERSION 1
#define SEL_ERR UINT64_MAX /* error sentinel for uint64_t-returning calls */

typedef enum {
  SEL_OK = 0,
  SEL_E_ARG = 1,       /* bad argument (null pointer, out-of-range index, bad sizes)            */
  SEL_E_ALIGN = 2,     /* column data pointer not 16-byte aligned                               */
  SEL_E_TYPE = 3,      /* unknown column type, or a constant not representable in its column   */
  SEL_E_PROGRAM = 4,   /* malformed predicate program (see "Program validation" below)          */
  SEL_E_TOO_LARGE = 5, /* global_rows >= 2^32 (row ids are uint32)                              */
  SEL_E_CUDA = 6,      /* CUDA runtime failure (message carries cudaGetErrorString)             */
  SEL_E_NCCL = 7,      /* NCCL failure or NCCL library not loadable                              */
  SEL_E_STATE = 8      /* call not valid in the context's state                                  */
} sel_status;

/* Column element types (PAPER.md:475-479 INTEGER, TEXT, DECIMAL(15,2); DATE at PAPER.md:681;
 * integer-coded dimension attributes at PAPER.md:725-726). Widths in bytes in brackets.
 *   SEL_INT32   [4]  signed two's complement
 *   SEL_INT64   [8]  signed two's complement (DECIMAL(15,2) as scaled cents)
 *   SEL_FLOAT32 [4]  IEEE-754 binary32; NaN compares false, -0 == +0
 *   SEL_DATE32  [4]  int32 days since 1970-01-01, compared as int32
 *   SEL_DICT8   [1], SEL_DICT16 [2], SEL_DICT32 [4]  unsigned dictionary codes of a sorted
 *               dictionary (code order == string order), compared as unsigned integers       */
typedef enum {
  SEL_INT32 = 1,
  SEL_INT64 = 2,
  SEL_FLOAT32 = 3,
  SEL_DATE32 = 4,
  SEL_DICT8 = 5,
  SEL_DICT16 = 6,
  SEL_DICT32 = 7
} sel_type;

/* One column of the local shard: `data` is a DEVICE pointer to local_rows elements of `type`,
 * 16-byte aligned, contiguous (columnar layout). dict_size is informational
 * for SEL_DICT* (codes >= dict_size simply never occur) and ignored otherwise. */
typedef struct {
  sel_type type;
  const void* data;
  uint32_t dict_size;
} sel_column;

typedef struct sel_ctx_s* sel_ctx;
typedef struct sel_table_s* sel_table;
typedef struct sel_prepared_s* sel_prepared;

/* ---- contexts ------------------------------------------------------------------------------
 * sel_ctx_create: binds to `cuda_device` (the caller's current device is not changed on return).
 *   Errors: SEL_E_ARG (null out), SEL_E_CUDA (bad device). */
sel_status sel_ctx_create(int cuda_device, sel_ctx* out);

/* sel_ctx_set_comm: make the context one rank of an `nranks`-GPU group (rows sharded
 * contiguously, one process per GPU). `nccl_unique_id` points to the 128-byte ncclUniqueId that
 * rank 0 produced with sel_nccl_unique_id and broadcast out of band (torch.distributed).
 * Collective: every rank must call it. NCCL is loaded with dlopen("libnccl.so.2") on first use.
 * nranks == 1 is allowed (a one-rank communicator). Errors: SEL_E_ARG, SEL_E_NCCL, SEL_E_STATE
 * (already set). Failure detection: while a probe waits for its stream the library polls
 * ncclCommGetAsyncError; an asynchronous NCCL error (a rank died) aborts the communicator and
 * fails the probe with SEL_E_NCCL instead of hanging, and every later probe of the context too. */
sel_status sel_ctx_set_comm(sel_ctx ctx, int nranks, int rank, const void* nccl_unique_id);

/* Cross-rank exchange over peer memory, without NCCL ("a one-shot peer write of each
 * rank's count into a symmetric buffer over NVLink plus a flag"). Each rank owns a small
 * symmetric buffer that every other rank maps through CUDA IPC; an exchange stores the rank's
 * counts (epoch-tagged) into every rank's buffer with system-scope release stores over
 * NVLink/NVSwitch and waits (acquire loads) until all ranks' values of that epoch arrived.
 * Once set, EVERY cross-rank combination of the context uses it instead of NCCL: sel_count's
 * sum (run by the count kernel's last CTA, fused with the count), sel_pushdown's offsets,
 * sel_count_batch / sel_count_sampled's sums, and sel_execute's one exchange per call — which
 * runs inside the count kernel's last CTA, right before the materialisation it gates, also in
 * prepared (graph) executes. A communicator is then not needed; if one is set as well, its
 * nranks/rank must agree.
 * sel_ctx_peer_handle: allocates the context's buffer (on first call) and writes its 64-byte
 *   CUDA IPC handle to out64 (host memory), to be shared out of band (torch.distributed).
 *   Errors: SEL_E_ARG, SEL_E_STATE (context destroyed), SEL_E_CUDA.
 * sel_ctx_set_peers: `handles` = nranks consecutive 64-byte handles, rank r's at 64*r (this
 *   rank's own entry is ignored). 1 <= nranks <= 32; the ranks may share a device (IPC maps
 *   a buffer of the same GPU too). Collective in effect: every rank must call it and then
 *   issue the same sequence of probes. A wait longer than the peer timeout (10 s unless
 *   sel_ctx_set_peer_timeout; a rank missing) makes the call fail with SEL_E_STATE instead of
 *   hanging. A failed exchange writes nothing: its gathered counts and sums are all-ones
 *   (UINT64_MAX), never a partial sum, so the gated push-down of an Execute (also one writing
 *   into another rank's buffers, sel_execute_to) stores no row. The failure is sticky: every
 *   later probe of the context fails with SEL_E_STATE until every rank drops its peers and sets
 *   them again (the ranks' exchange epochs are out of step).
 *   nranks == 0 drops the peers again (unmaps the others' buffers; handles may be NULL) — e.g.
 *   when not every rank could map every buffer and all fall back to a communicator; every rank
 *   should drop its peers before any rank destroys its context. Dropping also resets the
 *   exchange (epoch 0, an empty buffer, no failure).
 *   Errors: SEL_E_ARG (bad ranks, disagreeing with the communicator), SEL_E_STATE (already
 *   set, or no handle exported yet), SEL_E_CUDA (cudaIpcOpenMemHandle failed). */
sel_status sel_ctx_peer_handle(sel_ctx ctx, void* out64);
sel_status sel_ctx_set_peers(sel_ctx ctx, int nranks, int rank, const void* handles);
/* The peer exchange's wait bound in milliseconds (1 .. 3,600,000; default 10,000): the failure
 * detection of SURVEY §5 for the library's own collective. Takes effect for the next probe
 * (prepared executes re-capture). Errors: SEL_E_ARG. */
sel_status sel_ctx_set_peer_timeout(sel_ctx ctx, uint64_t timeout_ms);

/* Gather to one rank over peer memory ("an optional gather-to-one-rank uses P2P
 * writes at the offset"). sel_ctx_export_buffer: a 72-byte handle (CUDA IPC handle of the
 * allocation holding dev_ptr + the 8-byte offset of dev_ptr in it) to hand to other ranks.
 * sel_ctx_import_buffer: maps such a handle (once per allocation; unmapped by
 * sel_ctx_set_peers(ctx, 0, ...) or sel_ctx_destroy) and returns the device pointer, usable by
 * this context's kernels (NVLink/NVSwitch for another GPU's memory). Errors: SEL_E_ARG,
 * SEL_E_CUDA. The exporter must not free the buffer while it is mapped elsewhere. */
sel_status sel_ctx_export_buffer(sel_ctx ctx, const void* dev_ptr, void* out_handle72);
sel_status sel_ctx_import_buffer(sel_ctx ctx, const void* handle72, void** out_dev_ptr);

/* Writes a fresh 128-byte ncclUniqueId into `out128` (call on rank 0 only). SEL_E_NCCL on
 * failure. */
sel_status sel_nccl_unique_id(void* out128);

/* Destroys the context: frees its device scratch and communicator at once. If tables are still
 * registered, the context struct is freed when the last of them is released (sel_table_release
 * stays valid) and probes on them fail with SEL_E_STATE. */
void sel_ctx_destroy(sel_ctx ctx);

/* Kernel timing (for bench.py's roofline): when enabled, every probe records CUDA events around
 * its device kernels on the caller's stream; sel_ctx_last_kernel_ms reports the last probe's
 * main-kernel duration in milliseconds (0 if timing is off). */
sel_status sel_ctx_set_timing(sel_ctx ctx, int enable);
sel_status sel_ctx_last_kernel_ms(sel_ctx ctx, float* ms);
/* Device time of the most recent count probe's kernel and of the most recent push-down's kernels
 * (ms; 0 if timing is off or none ran). */
sel_status sel_ctx_last_times(sel_ctx ctx, float* count_ms, float* pushdown_ms);

/* ---- tables --------------------------------------------------------------------------------
 * sel_table_register: records descriptors of `ncols` (1..255) columns that
 * hold rows [global_row_offset, global_row_offset + local_rows) of a table with global_rows rows.
 * The descriptors are copied; the column memory must stay alive and unmodified while the table
 * exists. No data moves.
 *   Errors: SEL_E_ARG (null cols/out, ncols 0 or > 255, null data with local_rows > 0,
 *           global_row_offset + local_rows > global_rows, dict_size above the code range),
 *           SEL_E_TYPE (unknown type), SEL_E_ALIGN (data not 16-byte aligned),
 *           SEL_E_TOO_LARGE (global_rows >= 2^32). */
sel_status sel_table_register(sel_ctx ctx, const sel_column* cols, uint32_t ncols,
                              uint64_t local_rows, uint64_t global_row_offset,
                              uint64_t global_rows, sel_table* out);
void sel_table_release(sel_table table);

/* ---- probes --------------------------------------------------------------------------------
 * sel_count: exact |{ i : P(row i) }| over the table's rows. With peers
 * or a communicator it is the sum over all ranks (one exchange: the peer-memory exchange fused
 * into the count kernel, or one 8-byte NCCL all-reduce) and every rank gets the global count. Enqueues on `cuda_stream` (a cudaStream_t; NULL = legacy default stream)
 * and blocks until the count is on the host (the optimizer needs the number).
 * `prog` is host memory, copied during the call.
 * Returns the count, or SEL_ERR (SEL_E_ARG, SEL_E_PROGRAM, SEL_E_TYPE, SEL_E_CUDA, SEL_E_NCCL). */
uint64_t sel_count(sel_table table, const void* prog, size_t prog_bytes, void* cuda_stream);

/* sel_count_async: the same count, enqueued on `cuda_stream` WITHOUT waiting: the global count
 * (uint64) lands in the DEVICE word *d_out when the stream reaches it (with peers or a
 * communicator after the exchange, also enqueued). No host synchronisation, so the call can be
 * captured into a caller's CUDA graph or several probes pipelined ("an async variant
 * that writes the count to a device pointer"). The context's scratch is reused by every probe:
 * enqueue a context's asynchronous and blocking probes on ONE stream (or synchronise between
 * streams). Keeps no selection. Errors (validation, launch): as sel_count, returned at once;
 * kernel faults surface at the caller's next synchronisation. */
sel_status sel_count_async(sel_table table, const void* prog, size_t prog_bytes, uint64_t* d_out,
                           void* cuda_stream);

/* sel_count_ex: sel_count with flags.
 *   SEL_KEEP_SELECTION: the probe also keeps its selection in the context's scratch (the local row
 *   mask, 1 bit per row, plus per-1024-row counts: n/8 + n/512 bytes). A following sel_pushdown of
 *   the SAME table with byte-identical program bytes then materialises from it without
 *   re-evaluating the predicate (materialise right after the count, reusing the scan
 *   just done on the GPU; Algorithm 1 always counts before it executes).
 *   keep_cols/nkeep (host array, may be NULL/0): the compound's projected columns — Algorithm 1
 *   knows them before it counts (ExtractPushDown returns conditions and columns, PAPER.md:374,
 *   408). Those that are predicate columns have their selected values kept too (in row order per
 *   1024-row chunk; at most 8 columns and 8 bytes per row), so the push-down copies them instead
 *   of reading them again; the others are gathered by the push-down. The kept selection stays
 *   valid until the next SEL_KEEP_SELECTION probe on this context or the release of the table;
 *   the columns must not change in between (the registration contract).
 *   Errors: as sel_count, plus SEL_E_ARG (unknown flag, keep column index >= ncols). */
#define SEL_KEEP_SELECTION 1u
uint64_t sel_count_ex(sel_table table, const void* prog, size_t prog_bytes, uint32_t flags,
                      const uint32_t* keep_cols, uint32_t nkeep, void* cuda_stream);

/* sel_execute: Algorithm 1's Execute(compound, isSPD = true, maxSize) in one
 * call: count with SEL_KEEP_SELECTION (environment SEL_KEEP_VALUES=1: also keeping the projected
 * predicate columns' values, as sel_count_ex's keep_cols), then if the
 * GLOBAL count > max_size "throw" — *out_materialized = 0, nothing is written, *out_local_count
 * and *out_global_offset are set to 0 — else materialise exactly like sel_pushdown (from the kept
 * selection) and set *out_materialized = 1. Returns the global count or SEL_ERR. Arguments as
 * sel_pushdown; out_materialized may be NULL. With peers or a communicator the call issues
 * exactly one collective, gated or not: an exchange (peer memory) or all-gather (NCCL) of the
 * per-rank counts, whose sum is the global count the gate compares and whose exclusive prefix
 * is *out_global_offset (every rank must call it). */
uint64_t sel_execute(sel_table table, const void* prog, size_t prog_bytes,
                     const uint32_t* proj_cols, uint32_t nproj, uint64_t max_size,
                     uint32_t* out_rowids, void* const* out_cols, uint64_t capacity_rows,
                     uint64_t* out_local_count, uint64_t* out_global_offset,
                     int* out_materialized, void* cuda_stream);

/* sel_execute_to: sel_execute whose outputs are the GLOBAL result — typically one rank's buffers
 * mapped by every rank (sel_ctx_import_buffer): each rank writes its selected rows at its offset
 * (the exclusive prefix of the per-rank counts, computed on the device from the Execute's one
 * exchange), so the rank-ordered, ascending result assembles in place through P2P stores of the
 * materialisation kernel itself — no gather step. capacity_rows is the GLOBAL capacity of the
 * buffers (rows past it are not written). Other arguments, outputs and errors as sel_execute;
 * every rank must call it. */
uint64_t sel_execute_to(sel_table table, const void* prog, size_t prog_bytes,
                        const uint32_t* proj_cols, uint32_t nproj, uint64_t max_size,
                        uint32_t* out_rowids, void* const* out_cols, uint64_t capacity_rows,
                        uint64_t* out_local_count, uint64_t* out_global_offset,
                        int* out_materialized, void* cuda_stream);

/* Prepared executes: the same Execute with every argument fixed, validated and canonicalised
 * once and — for a program that scans a non-empty shard — its device work (count keeping the
 * selection, device-side gate, materialisation, result copies; with a communicator also the
 * count all-reduce and the all-gather of per-rank counts, NCCL operations being capturable;
 * environment SEL_GRAPH_COMM=0 leaves those uncaptured) captured into a CUDA graph, so
 * that a repeated probe (the optimizer re-estimating) costs one graph launch
 * and one synchronisation. The graph reads the columns' CURRENT contents at every run.
 * sel_prepare_execute: arguments as sel_execute (host arrays are copied; device buffers must
 * stay valid while prepared). Errors: as sel_execute's validation (SEL_E_ARG, SEL_E_PROGRAM,
 * SEL_E_TYPE, SEL_E_STATE), SEL_E_CUDA (capture).
 * sel_prepared_execute: one Execute on `cuda_stream`, blocking; outputs and return as
 * sel_execute. A run after the context reallocated its scratch (a probe of a larger table) or
 * after the bitmap registry changed re-captures first (SEL_E_ARG if a bitmap id the program
 * uses is no longer registered). SEL_E_STATE if the table was released.
 * sel_prepared_execute_async: the same Execute, returning as soon as its count — the number
 * Algorithm 1 decides on — and the outputs below are final on the host,
 * while the gated materialisation (Execute's temp table) is still running on
 * `cuda_stream`: the output buffers are valid once that stream reaches the point of the call
 * (order later work on it, or synchronise it). The last CTA of the work that finishes the count
 * stores the result words and then a sequence word into pinned host memory; the call spins on
 * that word (polling the stream for errors, and NCCL's asynchronous error with a communicator).
 * With per-kernel timing on (sel_ctx_set_timing), more than 512 ranks, or an uncaptured
 * execute (constant program, empty shard, SEL_GRAPH_COMM=0 with NCCL), it blocks like
 * sel_prepared_execute. The context's later calls reuse its selection and scratch buffers, which
 * the materialisation may still be reading: a call on another stream is ordered after it by the
 * library (an event wait), except while that stream is being captured into the caller's own CUDA
 * graph, where ordering it is the caller's part.
 * Errors: as sel_prepared_execute; SEL_E_STATE if the stream drained
 * without the Execute's result words; an error of the materialisation itself surfaces at the
 * caller's next synchronisation of the stream or the context's next call.
 * sel_prepared_release: frees the handle (NULL is a no-op); release it before its context. */
sel_status sel_prepare_execute(sel_table table, const void* prog, size_t prog_bytes,
                               const uint32_t* proj_cols, uint32_t nproj, uint64_t max_size,
                               uint32_t* out_rowids, void* const* out_cols,
                               uint64_t capacity_rows, sel_prepared* out);
uint64_t sel_prepared_execute(sel_prepared prepared, uint64_t* out_local_count,
                              uint64_t* out_global_offset, int* out_materialized,
                              void* cuda_stream);
uint64_t sel_prepared_execute_async(sel_prepared prepared, uint64_t* out_local_count,
                                    uint64_t* out_global_offset, int* out_materialized,
                                    void* cuda_stream);
void sel_prepared_release(sel_prepared prepared);

/* sel_pushdown: materialise sigma_P pi_proj(R) for the local shard.
 *   out_rowids : device uint32[capacity_rows], receives GLOBAL row ids (global_row_offset + i)
 *                of the selected local rows in ascending order.
 *   out_cols[j]: device buffer of capacity_rows elements of column proj_cols[j]'s type;
 *                out_cols[j][k] = column proj_cols[j] at row out_rowids[k] - global_row_offset.
 *   proj_cols  : host array of nproj column indices (< ncols; repeats allowed); nproj may be 0.
 *   Capacity gate (Algorithm 1): the call always computes the exact count;
 *   if the local count exceeds capacity_rows, exactly the first capacity_rows selected rows
 *   (ascending) are written and nothing beyond. This is not an error; the caller compares
 *   *out_local_count with its capacity ("throw" -> revert).
 *   out_local_count (host, may be NULL): selected rows in this shard.
 *   out_global_offset (host, may be NULL): exclusive prefix of the per-rank counts in rank order
 *   (0 with one rank) = this shard's position in the global ascending result.
 * Returns the global count (sum over ranks), or SEL_ERR. Blocks like sel_count.
 * Errors: as sel_count, plus SEL_E_ARG for a bad projection index or null outputs with
 * capacity_rows > 0. */
uint64_t sel_pushdown(sel_table table, const void* prog, size_t prog_bytes,
                      const uint32_t* proj_cols, uint32_t nproj, uint32_t* out_rowids,
                      void* const* out_cols, uint64_t capacity_rows, uint64_t* out_local_count,
                      uint64_t* out_global_offset, void* cuda_stream);

/* Which path the context's last sel_pushdown took: 1 = from a kept selection (no predicate
 * evaluation, no look-back), 2 = two passes inside the call (a count keeping the selection and
 * the projected predicate columns' values, then path 1's materialisation; taken without a kept
 * selection when the shard has >= 3·2^20 rows), 0 = single pass (evaluate + decoupled look-back;
 * smaller shards), -1 = no kernel ran (empty shard or constant-false program). Environment, read
 * at sel_ctx_create: SEL_PUSHDOWN_PATH=single forces the single pass, =two the two passes;
 * SEL_TWO_PASS_MIN_ROWS=<n> moves the threshold. Path 2 leaves its selection kept, so a repeated
 * sel_pushdown of the same program takes path 1. */
int sel_ctx_last_pushdown_path(sel_ctx ctx);

/* How the context's last materialisation from a kept selection (path 1 or 2 above, also inside
 * sel_execute) wrote its projections — diagnostics and tests, no effect on results. Bits:
 * SEL_PD_CODED (a projection written from the kept code bits of a two-point leaf, the column not
 * read), SEL_PD_WHOLE_CHUNKS (fully selected 1024-row chunks left to the whole-chunk copy kernel),
 * SEL_PD_CONSTANT (a projection pinned to one value by the conjunction, filled), SEL_PD_KEPT_VALUES
 * (a projection copied from values the count kept). 0 for other paths; -1 for a null ctx. */
#define SEL_PD_CODED 1
#define SEL_PD_WHOLE_CHUNKS 2
#define SEL_PD_CONSTANT 4
#define SEL_PD_KEPT_VALUES 8
int sel_ctx_last_pushdown_flags(sel_ctx ctx);

/* Choose the path sel_pushdown takes when no kept selection matches (overrides the environment
 * above): mode -1 = automatic (two passes at >= 3·2^20 local rows, else the single pass), 0 = always
 * the single pass (also for sel_execute, which then gates on the host: count, then single pass),
 * 2 = always two passes. A matching kept selection is used in every mode but 0.
 * Errors: SEL_E_ARG (null ctx, other mode). */
sel_status sel_ctx_set_pushdown_path(sel_ctx ctx, int mode);

/* sel_count_batch: exact counts of nprog (1..32) programs over the table in
 * ONE scan — each referenced column is read once per chunk and each distinct leaf (same column and
 * same canonical interval set, across programs) evaluated once. out_counts: host array of nprog,
 * global over ranks (one all-reduce of nprog u64). Limits after canonicalisation: <= 32 distinct
 * leaves, <= 32 columns, <= 1024 intervals, <= 512 postfix ops in total, no IN_BITMAP leaves
 * (else SEL_E_ARG).
 * Errors: as sel_count. Blocks until the counts are on the host. */
sel_status sel_count_batch(sel_table table, const void* const* progs, const size_t* prog_bytes,
                           uint32_t nprog, uint64_t* out_counts, void* cuda_stream);

/* Bitmaps for IN_BITMAP leaves: `words` is a DEVICE array of
 * ceil(nbits/64) uint64 (16-byte aligned, caller-owned, alive and unmodified while registered);
 * bit i (word i/64, bit i%64) = key i is in the set. nbits < 2^31. Ids are small integers, valid
 * for the context until released. Errors: SEL_E_ARG, SEL_E_ALIGN, SEL_E_TOO_LARGE (too many). */
sel_status sel_bitmap_register(sel_ctx ctx, const uint64_t* words, uint64_t nbits,
                               uint32_t* out_id);
sel_status sel_bitmap_release(sel_ctx ctx, uint32_t id);

/* sel_count_sampled: the exact count over a BLOCK SAMPLE of the table —
 * the 1024-row chunks c with c mod stride == phase (stride >= 1, phase < stride; stride 1 is the
 * whole table) — for the sampling estimator |sigma(R')| * |R| / |R'| of PAPER.md:199-203, shown
 * beside the exact probe. *out_sample_rows (may be NULL) receives |R'|. Global over ranks.
 * Returns the sample's count or SEL_ERR (SEL_E_ARG for a bad stride/phase; as sel_count). */
uint64_t sel_count_sampled(sel_table table, const void* prog, size_t prog_bytes, uint32_t stride,
                           uint32_t phase, uint64_t* out_sample_rows, void* cuda_stream);

/* sel_histogram (a synopsis baseline beside the exact probe): an EQUI-DEPTH
 * histogram of column `col` over the same block sample as sel_count_sampled
 * (chunks c mod stride == phase; stride 1 = every row), local shard only. The sample's m values
 * are sorted (CUB radix sort on the device) and cut into nbuckets (1..65536) buckets of
 * positions [floor(b m / B), floor((b+1) m / B)); bucket b reports its lowest and highest value
 * (out_lo/out_hi, the column's values as int64), its rows (out_rows) and its number of distinct
 * values V(b) (out_distinct) — host arrays of nbuckets; an empty bucket (m < B) reports
 * lo = hi = 0, rows = distinct = 0. *out_sample_rows (may be NULL) = m. The
 * paper's equality estimate |sigma_{A=x}(R)| = D / V(b_x), D = T(R) / B, over these arrays is
 * sel_equi_depth_estimate below.
 * Errors: SEL_E_ARG (bad stride/phase/nbuckets/column), SEL_E_TYPE (not INT32/DATE32/DICT*),
 * SEL_E_TOO_LARGE (a sample of >= 2^31 rows), SEL_E_CUDA. */
sel_status sel_histogram(sel_table table, uint32_t col, uint32_t stride, uint32_t phase,
                         uint32_t nbuckets, int64_t* out_lo, int64_t* out_hi, uint64_t* out_rows,
                         uint64_t* out_distinct, uint64_t* out_sample_rows, void* cuda_stream);

/* The synopsis estimators themselves (host arithmetic, no device work):
 * sel_sample_estimate: the sampling estimator |sigma(R')| * |R| / |R'| of a
 *   block-sample count (sel_count_sampled): sample_count * table_rows / sample_rows, computed in
 *   double; 0 when sample_rows is 0.
 * sel_equi_depth_estimate: the equi-depth equality estimate |sigma_{A=x}(R)| = D / V(b_x) with
 *   D = table_rows / nbuckets, summed over EVERY bucket b whose [lo_b, hi_b]
 *   holds x and V(b) > 0 (the reading under which the paper's "30/2 + 30/1 + 30/7 = 49.3" follows
 *   the formula). lo/hi/distinct: sel_histogram's host arrays of nbuckets.
 *   Returns the estimate; NaN for null arrays or nbuckets 0. */
double sel_sample_estimate(uint64_t sample_count, uint64_t sample_rows, uint64_t table_rows);
double sel_equi_depth_estimate(const int64_t* lo, const int64_t* hi, const uint64_t* distinct,
                               uint32_t nbuckets, uint64_t table_rows, int64_t value);

/* Validate a program against column types without running it (host only; no GPU needed).
 * Returns SEL_OK or the status sel_count would report for it. */
sel_status sel_program_check(const void* prog, size_t prog_bytes, const sel_type* types,
                             uint32_t ncols);

/* Which device path a program takes after canonicalisation: 0 = generic interpreter,
 * 1 = conjunctive interval fast path, 2 = constant (folded to TRUE/FALSE, no scan needed);
 * negative status on error. Host only. */
int sel_program_path(const void* prog, size_t prog_bytes, const sel_type* types, uint32_t ncols);

/* The canonical plan the device would execute, as JSON, for host-side inspection and tests:
 *   {"path": p, "const": b, "max_depth": d,
 *    "ops": [[opcode, arg], ...],              opcode 0 = leaf(arg), 1 = AND, 2 = OR (postfix)
 *    "leaves": [{"col": c, "wclass": w, "fkey": f, "lo": [...], "span": [...]}, ...],
 *    "fast": [k, ...]}                          the count kernel's fast-path leaf kinds, one per
 *                                               leaf (0 point/4 B, 1 interval/4 B, 2 <= 4
 *                                               intervals/4 B, 3 interval/8 B, 4 <= 4 points/1 B),
 *                                               or [] when the interpreter runs the program
 * lo/span are the packed device values: a row value v (its raw bits, zero-extended; FLOAT32
 * first mapped through the sortable key) lies in the leaf iff ((v - lo) mod 2^W) <= span for
 * some interval, W = 64 for 8-byte columns and 32 otherwise. Writes at most `cap` bytes
 * (NUL-terminated when it fits) and returns the full length, or -status on a bad program. */
long sel_program_plan_json(const void* prog, size_t prog_bytes, const sel_type* types,
                           uint32_t ncols, char* buf, size_t cap);

sel_status sel_last_error(void);
const char* sel_last_error_message(void);
int sel_abi_version(void);

/* ==== Program byte format, version 1 (little-endian) ==========================================
 *
 * A predicate program is postfix code over a boolean stack (the paper's predicates are AND/OR
 * combinations of column-vs-constant comparisons).
 *
 *   header   12 B : u32 magic = bytes "SELP" | u16 version = 1 | u16 n_instr | u16 n_consts
 *                   | u16 reserved = 0
 *   n_instr x 8 B : u8 op | u8 col | u16 a | u16 b | u16 reserved = 0
 *   n_consts x 8 B: u64 constant slots
 *
 * Constant slots hold a value in the type of the column it is compared with:
 *   INT32, DATE32 : the int32 value sign-extended to 64 bits
 *   INT64         : the raw 64-bit value
 *   FLOAT32       : the binary32 bit pattern in the low 32 bits, high 32 bits zero
 *   DICT8/16/32   : the code zero-extended (must be < 2^8, 2^16, 2^32 respectively)
 *
 * Opcodes (v = the column `col` value of the current row; k[i] = constant slot i):
 *   0x01 TRUE                  push true          (col, a, b must be 0)
 *   0x02 FALSE                 push false         (col, a, b must be 0)
 *   0x10 EQ  push v == k[a]    0x11 LT push v < k[a]    0x12 GT push v > k[a]
 *   0x13 LE  push v <= k[a]    0x14 GE push v >= k[a]   (b must be 0)
 *   0x20 BETWEEN               push k[a] <= v && v <= k[b]  (inclusive; empty if k[a] > k[b])
 *   0x30 IN                    push v == k[a] || ... || v == k[a+b-1]   (1 <= b <= 256)
 *   0x31 IN_BITMAP             push 0 <= v < nbits(a) && bit v of bitmap a is set, where a is an
 *                              id from sel_bitmap_register (b must be 0; integer columns only) —
 *                              a dimension-derived key set pushed onto a foreign key (SURVEY §8f
 *                              NEXT(3); e.g. SSB `s_region = 1` as a set of lo_suppkey values)
 *   0x40 AND, 0x41 OR          pop y, pop x, push x AND/OR y      (col, a, b must be 0)
 *   0x42 NOT                   pop x, push NOT x                  (col, a, b must be 0)
 * Comparisons use the column type's order: signed for INT32/INT64/DATE32, unsigned for DICT*,
 * IEEE-754 for FLOAT32 (any comparison with NaN is false; -0 == +0). Logic is two-valued (no
 * NULLs). The row is selected iff the single value left on the stack is true.
 *
 * Program validation (first failing check wins, in this order):
 *   1. prog_bytes < 12, magic != "SELP", version != 1, n_instr == 0, n_instr > 128,
 *      n_consts > 512, header reserved != 0, or prog_bytes != 12 + 8*(n_instr + n_consts)
 *      -> SEL_E_PROGRAM.
 *   2. For each instruction in order:
 *      a. reserved != 0, unknown op                                          -> SEL_E_PROGRAM
 *      b. TRUE/FALSE/AND/OR/NOT with col, a or b nonzero                      -> SEL_E_PROGRAM
 *      c. comparison/BETWEEN/IN/IN_BITMAP: col >= ncols; EQ..GE with b != 0 or a >= n_consts;
 *         BETWEEN with a or b >= n_consts; IN with b == 0, b > 256 or a + b > n_consts;
 *         IN_BITMAP with b != 0                                               -> SEL_E_PROGRAM
 *      d. stack underflow (AND/OR need 2, NOT needs 1), or depth after the instruction > 16
 *                                                                             -> SEL_E_PROGRAM
 *      e. a referenced constant slot not representable in the column's type, or
 *         IN_BITMAP on a FLOAT32 column                                       -> SEL_E_TYPE
 *   (whether an IN_BITMAP id is registered is checked by the probe: SEL_E_ARG)
 *   3. stack depth after the last instruction != 1                            -> SEL_E_PROGRAM
 * Maximum program size: 12 + 8 * (128 + 512) = 5,132 bytes.
 */

/* sel_ctx_set_option: the tuning switches below, per context (the environment variables only
 * give their initial values at sel_ctx_create). None of them changes a result, only which kernel
 * variant or launch shape produces it. Setting one drops the context's kept selection and makes
 * prepared executes re-capture. Names and values:
 *   "fast" 0|1, "coded" 0|1, "dense_split" 0|1, "keep_values" 0|1, "graph_comm" 0|1,
 *   "prefetch" -1 (auto) | 0 | 1, "count_warps" 0 (auto) | 8, "two_pass_min_rows" n >= 0
 *   (ignored while sel_ctx_set_pushdown_path forces the single pass), "ctas_per_sm" 0 (the
 *   occupancy calculator's) | k. Errors: SEL_E_ARG (null, unknown name, value out of range),
 *   SEL_E_STATE (context destroyed). */
sel_status sel_ctx_set_option(sel_ctx ctx, const char* name, int64_t value);

/*
 * Environment (read once, by sel_ctx_create, as the initial values of sel_ctx_set_option's
 * switches; for A/B measurement and diagnosis — none of them changes a result, only which kernel
 * variant or launch shape produces it; DESIGN.md §5-§7 gives the measurements behind each
 * default):
 *   SEL_FAST=0               conjunctions through the postfix interpreter, not the fast path
 *   SEL_CODED=0              no coded projections (two-point columns read by the push-down)
 *   SEL_DENSE_SPLIT=0        no whole-chunk copy kernel for fully selected chunks
 *   SEL_KEEP_VALUES=1        the keeping count also keeps projected predicate columns' values
 *   SEL_PREFETCH=0|1         force the count's L2 bulk prefetch of the next chunk off / on
 *   SEL_GRAPH_COMM=0         no cross-rank collective inside prepared (graph) executes
 *   SEL_PUSHDOWN_PATH=single|two   sel_pushdown always single-pass / always two passes
 *   SEL_TWO_PASS_MIN_ROWS=n  shard size from which sel_pushdown takes two passes (3*2^20)
 *   SEL_COUNT_NW=8           8-warp count CTAs even when staged key sets allow 32
 *   SEL_CTAS_PER_SM=k        cap the count kernels' resident CTAs per SM (grid = 148 * k)
 */

#ifdef __cplusplus
}
#endif
#endif /* SEL_H_ */
