/*
 * bdlora.h -- C ABI of the B200-native BD-LoRA tensor-parallel multi-adapter LoRA layer.
 *
 * Paper: "Block-diagonal LoRA" (BD-LoRA), arXiv 2510.23346 (PAPER.md, cited as P:<line>).
 *
 * The layer, per token t with adapter a(t) from a resident pool:
 *
 *     y_t = x_t W + s_a * (x_t A_a) B_a
 *
 * sharded Megatron-style over N = tp_size devices:
 *   column-parallel (QKV, gate|up):  W, A column-sharded, B BLOCK-DIAGONAL   (Alg. 2)
 *   row-parallel    (O, down):       W row-sharded, A BLOCK-DIAGONAL, B row-sharded, one all-reduce
 *                                    of the base+LoRA partial                 (Alg. 1)
 * so BD-LoRA adds ZERO collectives.  The S-LoRA sharding is provided as the comparison
 * path: +1 all-gather per column layer, +1 all-reduce per row layer.
 *
 * Conventions (all entry points):
 *   - Every function returns a bdlora_status; on failure bdlora_last_error() (thread-local) names
 *     the offending argument / shape / value.  No C++ exception crosses this boundary.
 *   - Tensors are plain pointers.  "device" pointers are CUDA device memory of the pool's device;
 *     bf16 = IEEE bfloat16 (uint16 storage), row-major, densely packed unless an ld is given.
 *   - Ownership: the caller owns X, W, Y, ids and the workspace; the library never frees them.
 *     The pool owns adapter memory.  The comm owns its ncclComm_t.
 *   - Streams: all device work is enqueued on `stream` (a cudaStream_t passed as void*, 0 = legacy
 *     default).  Forward calls do no allocation, no host synchronisation and no device-side
 *     validation, so they are CUDA-graph capturable.  Validation is on host-side shapes only;
 *     asynchronous CUDA faults surface on a later call as BDLORA_E_CUDA.
 *   - ids contract: ids[t] in [-1, capacity) and referring to a LOADED slot; -1 = no adapter
 *     (LoRA term exactly 0, reading R8).  Not checked on device.
 *   - A pool is not thread-safe; distinct pools / devices are independent.
 *   - Numerics (reading R7): bf16 inputs, fp32 accumulation, the LoRA intermediate
 *     v = s * x A is kept in fp32 (also for the S-LoRA collective payloads), the base and LoRA
 *     terms are summed in fp32 and rounded to bf16 ONCE (RNE).  Row partials are rounded to bf16
 *     before the bf16 all-reduce.
 *   - N == 1: BD == S-LoRA == plain LoRA, no NCCL call is made.  T == 0: no-op (BDLORA_OK).
 *   - Layout deviation (documented in DESIGN.md): the paper writes W in R^{d_in x d_out}; the
 *     ABI takes W^T, i.e. [d_out_loc, d_in_loc] row-major ("nn.Linear.weight" / K-major), which makes
 *     both tensor-core operands K-major.  Adapter factors are given in the paper's orientation.
 *
 * Build: sm_100a only (-gencode arch=compute_100a,code=sm_100a); other devices -> BDLORA_E_ARCH.
 */
#ifndef BDLORA_H_
#define BDLORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BDLORA_ABI_VERSION 1
#define BDLORA_UNIQUE_ID_BYTES 128
#define BDLORA_MAX_SLICES 3

typedef struct bdlora_pool bdlora_pool; /* opaque: one per (device, projection, sharding mode)  */
typedef struct bdlora_comm bdlora_comm; /* opaque: wraps an ncclComm_t owned by the library      */
typedef struct bdlora_peer bdlora_peer; /* opaque: peer-mapped receive buffers of the fused AR  */
typedef void* bdlora_stream_t;          /* cudaStream_t                                          */

typedef enum {
  BDLORA_OK = 0,
  BDLORA_E_ARG = 1,          /* null pointer, negative size, shape mismatch, bad enum          */
  BDLORA_E_DIVISIBILITY = 2, /* d_in / d_out / rank not divisible by tp_size          */
  BDLORA_E_CAPACITY = 3,     /* slot out of range, rank > max_rank, arena full, T too large     */
  BDLORA_E_NOT_LOADED = 4,   /* slot not loaded (unload / host-side checks)                     */
  BDLORA_E_MODE = 5,         /* BD pool passed to slora_* or vice versa, row pool to column fn  */
  BDLORA_E_CUDA = 6,         /* CUDA runtime error (message has cudaGetErrorString)             */
  BDLORA_E_NCCL = 7,         /* NCCL error                                                      */
  BDLORA_E_ARCH = 8          /* device is not sm_100 (compute capability 10.0)                  */
} bdlora_status;

enum { BDLORA_COLUMN = 0, BDLORA_ROW = 1 };
/* BD-LoRA; S-LoRA; NFS-LoRA = A_1 and B_2 replicated, a full copy on every
   device (same collectives as BD-LoRA, N x the memory and compute for A_1 and B_2).       */
enum { BDLORA_SHARD_BD = 0, BDLORA_SHARD_SLORA = 1, BDLORA_SHARD_NFS = 2 };

typedef struct {
  int32_t parallel;   /* BDLORA_COLUMN | BDLORA_ROW                                              */
  int32_t sharding;   /* BDLORA_SHARD_BD | BDLORA_SHARD_SLORA | BDLORA_SHARD_NFS                 */
  int32_t tp_size;    /* N >= 1                                                                  */
  int32_t tp_rank;    /* i in [0, N): block i lives on device i (reading R2)          */
  int32_t d_in;       /* FULL input dim                                                          */
  int32_t n_slices;   /* J: 1; 2 = gate|up; 3 = q|k|v (each slice has its own A, B; reading R4).
                         ROW requires 1.                                                         */
  int32_t d_out[BDLORA_MAX_SLICES]; /* FULL output dim per slice                                 */
  int32_t capacity;   /* resident adapter slots (ids index these)                                */
  int32_t max_rank;   /* full-rank bound r_max; BD / S-LoRA column require tp_size | every rank  */
  int64_t arena_bytes;/* 0 = capacity x max_rank sizing; else a ragged first-fit arena of this size*/
} bdlora_pool_desc;

/* ---------------------------------------------------------------- library / device ---------- */
int bdlora_abi_version(void);
const char* bdlora_last_error(void); /* thread-local, never NULL; "" when no error            */
/* BDLORA_OK iff `cuda_device` is sm_100 (CC 10.0) and the library's kernels can run on it.     */
int bdlora_device_check(int cuda_device);
/* Number of kernels this library has enqueued since it was loaded (host-side count of launches;
   a CUDA-graph replay re-runs the captured launches without counting them again).              */
int bdlora_kernel_launches(int64_t* n);
/* Programmatic dependent launch chaining (default ON): every kernel of a forward is launched with
   programmatic stream serialization and waits (griddepcontrol.wait) before reading anything the
   preceding kernel may have produced (X, ids, v) and before writing Y, so a forward's prologue and
   weight stream overlap the tail of the preceding kernel.  Contract while ON: the base weight W, the
   pool's adapter factors and slot table, and the ids array must not be written by the KERNEL
   immediately preceding a forward on the same stream (the decode kernel streams W and reads ids, the
   slot entries and the adapters' B rows before the dependency resolves; X and v are read after it).
   Copies, memsets and event waits before a forward are full dependencies and are always safe.
   0 = plain stream order.                                                                         */
int bdlora_set_pdl(int enable);
/* Decode (T <= 16) LoRA schedule inside the fused single-kernel forward.  The layer is linear in a
   partition of K (y = sum_seg X_seg W_seg + s (X_seg A_seg) B, regrouping matmul_3/4 and matmul_5/6 of
   Alg. 1/2), so each CTA streaming a K-range of W can add its own share of the LoRA term:
   0 = GLOBAL: v = s X A computed once by the grid, every CTA waits for the whole v before its expand;
   1 = AUTO (default): K-local when the token tile holds ONE adapter group of rank <= 16 on this
       device, the tiles are reduced through a thread-block cluster and every CTA's K segment is
       short (<= 8 k-blocks, env BDLORA_LOCAL_MAXKB) -- the A rows then ride the weight pipeline as a
       16-row TMA box per stage and a second tcgen05 MMA accumulates v_seg; else GLOBAL;
   2 = same eligibility as 1 (kept for compatibility).  Results agree to fp32 summation order.
   Also settable with the environment variable BDLORA_LOCAL.  E_ARG for other values.                */
int bdlora_set_decode_lora(int mode);
/* Schedule knobs read once per process from the environment.  They change scheduling only, never values
   (tests/test_gpu_env_variants.py re-runs the parity tests under each); the defaults are the measured best:
     BDLORA_CLUSTER=0         split-K partials through global memory instead of a thread-block cluster
     BDLORA_CLUSTER_SHRINK=0  keep the split when its clusters do not fit one wave (global fix-up)
     BDLORA_STREAMK_CTAS=n    CTAs of a stream-K launch (default: whole tiles per CTA, else 0.86 x #SM)
     BDLORA_FUSED_MAX_T=n     largest batch served by the single-kernel forward (default 16, max 256)
     BDLORA_TC_EXPAND=0       LoRA expand on the CUDA cores for T > 16 too
     BDLORA_LOCAL / BDLORA_LOCAL_MAXKB   see bdlora_set_decode_lora
     BDLORA_STAGES=n          cap on the weight-ring depth;  BDLORA_GRID_CAP=n  cap on the SMs used
     BDLORA_DEBUG=1           print the cluster / split decisions to stderr                            */
/* Profiling hook: if non-NULL, subsequent tensor-core GEMM launches record per-CTA %globaltimer
   stamps (32 int64 per CTA) into this device buffer (>= 148*32*8 bytes); NULL turns it off.      */
int bdlora_debug_trace(void* device_buffer);

/* ---------------------------------------------------------------- communicator (NCCL) ------- */
/* NCCL 2.28 over NVLink/NVSwitch.  Bootstrap: rank 0 calls bdlora_comm_unique_id, the caller
   broadcasts the 128 bytes (e.g. torch.distributed.broadcast), every rank calls bdlora_comm_init. */
int bdlora_comm_unique_id(uint8_t id[BDLORA_UNIQUE_ID_BYTES]);
int bdlora_comm_init(const uint8_t id[BDLORA_UNIQUE_ID_BYTES], int nranks, int rank, int cuda_device,
                     bdlora_comm** out);
int bdlora_comm_destroy(bdlora_comm* comm);
/* Collective call log since init (SPEC S:148 per-tag counters):
   counts[0] base all-reduce calls, [1] LoRA all-gather calls, [2] LoRA all-reduce calls,
   [3] base all-reduce bytes, [4] LoRA all-gather bytes (per rank, sent), [5] LoRA all-reduce bytes.
   BD-LoRA paths never touch counts[1], [2], [4], [5] (Fig. 3 caption).               */
int bdlora_comm_stats(const bdlora_comm* comm, int64_t counts[6]);

/* ---------------------------------------------------------------- fused row all-reduce ------ */
/* the row-parallel layer's base all-reduce (Alg. 1 line 15) fused with
   the GEMM.  A peer group maps every rank's receive buffer ([2 parities][N sources][max_elems] fp32) and
   arrival counters into every rank's address space (CUDA IPC over NVLink / NVSwitch).  The decode kernel's
   epilogue writes its fp32 row partial P_i straight into slot [parity][i] of EVERY rank's buffer (peer
   stores, tile by tile as the tiles finish) and each CTA then signals every rank with a system-scope
   release; a small reduce kernel on each rank waits for N x grid arrivals and sums the N slots IN RANK
   ORDER in fp32, rounding once to bf16 -- every rank gets the same bits, and the sum is more accurate
   than the bf16 NCCL reduction of bdlora_row_forward (reading R7: rounding once).  No NCCL launch.
   Decode batches only (T <= 16 with the decode kernel's K-local LoRA capacity; else E_CAPACITY: use
   bdlora_row_forward).  BD and NFS row pools (S-LoRA keeps its NCCL collectives: E_MODE).
   Calls on one peer group must be issued in the same order on every rank (call parity alternates);
   push and reduce of one rank must not be separated by another push on the same group.                */
/* Collective over `comm` (every rank calls it): allocates this rank's buffers (2 x nranks x max_elems
   fp32; max_elems >= T x d_out of any call) and exchanges IPC handles through the communicator.        */
int bdlora_peer_create(bdlora_comm* comm, int64_t max_elems, bdlora_peer** out);
/* Test / emulation: `nranks` peer groups of one process on ONE device (out[r] = rank r), mapping each
   other's buffers directly.  Issue every rank's push before any rank's reduce (a reduce that waits for a
   push queued behind it on the same stream would spin; after ~2 s it gives up and flags an error).     */
int bdlora_peer_create_local(int nranks, int cuda_device, int64_t max_elems, bdlora_peer** out);
int bdlora_peer_destroy(bdlora_peer* peer);
/* 1 if a reduce gave up waiting for peers (~2 s), else 0 (synchronises the device).                   */
int bdlora_peer_error(const bdlora_peer* peer, int32_t* err);
/* Phase 1: P_i = X_i W_i + s (X_i A_i[a]) B_i[a] (Alg. 1 lines 9-12) computed by the decode kernel and
   pushed, fp32, into every rank's receive slot.  X [T, d_in/N], W = W_i^T [d_out, d_in/N], ids [T].    */
int bdlora_row_partial_push(bdlora_pool* pool, bdlora_peer* peer, const void* X, int64_t T, const void* W,
                            const int32_t* ids, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
/* Phase 2: Y [T, M] bf16 = sum over ranks of the pushed partials (M = d_out), once all have arrived.     */
int bdlora_peer_reduce(bdlora_peer* peer, void* Y, int64_t T, int32_t M, bdlora_stream_t stream);
/* Both phases: Y = AllReduce_i(P_i), replicated on every rank (Alg. 1 end to end).         */
int bdlora_row_forward_fused(bdlora_pool* pool, bdlora_peer* peer, const void* X, int64_t T, const void* W,
                             const int32_t* ids, void* Y, void* workspace, size_t ws_bytes,
                             bdlora_stream_t stream);

/* ---------------------------------------------------------------- adapter pool -------------- */
int bdlora_create_pool(const bdlora_pool_desc* desc, int cuda_device, bdlora_pool** out);
int bdlora_destroy_pool(bdlora_pool* pool);

/* Copies the FULL (unsharded) factors of one adapter and keeps only device tp_rank's shard
   ("modified the slicing code"), stored compactly -- no zero of a block-diagonal
   factor is stored or touched.  A[j], B[j] are bf16, paper orientation, row-major:
     COLUMN + BD   : A[j] d_in x r ;  B[j] compact (r/N) x d_out[j], the N diagonal blocks
                     (r/N) x (d_out[j]/N) side by side
     ROW    + BD   : A[0] compact d_in x (r/N), the N diagonal blocks (d_in/N) x (r/N) stacked
                      ;  B[0] r x d_out
     *      + SLORA: dense A[j] d_in x r ;  B[j] r x d_out[j]
     *      + NFS  : dense A[j] d_in x r ;  B[j] r x d_out[j]; the device keeps A_1 whole and B_1's
                     column block i (COLUMN), A_2's row block i and B_2 whole (ROW)
   rank r: 1 <= r <= max_rank, BD needs N | r (else BDLORA_E_DIVISIBILITY).  scale = s_a applied to
   the fp32 shrink output (e.g. alpha*sqrt(N)/sqrt(r) for BD; reading R1).  src_is_device:
   0 = host pointers (copied synchronously w.r.t. `stream`; sources may be freed on return),
   1 = device pointers (caller may free after `stream` completes).  Reloading a loaded slot
   replaces it; no forward that reads the slot may be in flight.  Ragged arena: the new copy is
   allocated and staged before the old one is released, so a failed reload (E_CAPACITY, E_CUDA)
   leaves the previous adapter loaded.  Fixed arena (arena_bytes = 0): the slot's own region is
   rewritten, so a copy failure leaves the slot empty (E_NOT_LOADED on later use of the id is the
   caller's contract, not checked on device).                                                    */
int bdlora_load_adapter(bdlora_pool* pool, int32_t slot, int32_t rank, float scale,
                        const void* const* A, const void* const* B, int32_t src_is_device,
                        bdlora_stream_t stream);
/* Downward-compatible BD serving: an adapter TRAINED for N_h = n_blocks
   devices (its compact B_1 / A_2 hold N_h diagonal blocks) served on tp_size = N_l devices, N_l | N_h.
   Device i runs the work of the N_h-layout devices i*m .. (i+1)*m - 1 (m = N_h/N_l) -- "stacking the
   computations of different devices": its A_1 / B_2 shards are the union of theirs (rank chunk
   [i r/N_l, (i+1) r/N_l)), and its local B_1 (COLUMN) or A_2 (ROW) is block-diagonal with those m
   blocks.  Only the blocks are stored and read: COLUMN B_1 as [r/N_h, d_out_j/N_l] (the m
   blocks side by side; the expand of block bb's columns reads v rows [bb r/N_h, (bb+1) r/N_h)), ROW A_2
   as [r/N_l, d_in/N_h] (rank row q holds the inputs of its block q / (r/N_h) only).  A pool holds one
   block count m: loading an adapter with another m while others are resident is E_MODE.  Pools with
   m > 1 run every batch through the multi-adapter decode kernels, in chunks of <= 64 tokens (the base
   weights are streamed once per chunk).  Load format = bdlora_load_adapter's BD format with N_h in place
   of N.  BD pools only (E_MODE); N_l | N_h, N_h | r and N_h | d_out[j] (COLUMN) or d_in (ROW); m > 1 also
   needs 128-column-aligned slices with blocks of a multiple of 8 columns (COLUMN) or 8 | d_in/N_h and
   64 | d_in/N_l (ROW) (E_DIVISIBILITY).  n_blocks == tp_size = bdlora_load_adapter.                  */
int bdlora_load_adapter_blocks(bdlora_pool* pool, int32_t slot, int32_t rank, float scale,
                               const void* const* A, const void* const* B, int32_t n_blocks,
                               int32_t src_is_device, bdlora_stream_t stream);
int bdlora_unload_adapter(bdlora_pool* pool, int32_t slot);
/* Resident adapter bytes (compact shards) and arena capacity in bytes.                          */
int bdlora_pool_bytes(const bdlora_pool* pool, int64_t* resident, int64_t* arena);
/* Local geometry: K_loc (input dim of X on this device) and M_loc (output columns on this
   device: sum_j d_out[j]/N for COLUMN, d_out[0] for ROW).                                        */
int bdlora_pool_geometry(const bdlora_pool* pool, int32_t* k_loc, int32_t* m_loc);

/* Workspace bytes needed by any forward of this pool for T tokens (device memory, caller-owned,
   256-byte aligned base).  The first 64 KB are a COUNTER REGION at T-independent offsets (split-tile
   arrival counters, the fused shrink's tickets): it must be ZERO before the workspace's first use
   (bdlora_workspace_init, or any zero fill such as cudaMemset of the whole buffer) and every forward
   leaves it zero again.  The rest is scratch, undefined on entry.  A workspace sized for T may then
   serve any T' <= T of this pool, one call at a time in stream order (calls on different streams
   need different workspaces).  An uninitialised counter region can make a forward spin or return a
   wrong split-K sum -- it is not detected.                                                       */
int bdlora_workspace_bytes(const bdlora_pool* pool, int64_t T, size_t* bytes);
/* Zeroes the workspace's counter region on `stream` (E_ARG if ws_bytes < 64 KB).                 */
int bdlora_workspace_init(const bdlora_pool* pool, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
/* Debug/test hook: the last tensor-core kernel launch made by the CALLING thread:
   info[0] instantiation (0 GEMM + expand, 1 tensor-core shrink, 2 single-kernel decode forward,
   3 lean decode forward), [1] token-tile width BN, [2] grid (CTAs), [3] cluster size, [4] ring stages,
   [5] 128-row tiles, [6] token tiles, [7] 64-wide k-blocks.  info[0] = -1 before any launch.      */
int bdlora_last_launch_info(int32_t info[8]);

/* ---------------------------------------------------------------- routing metadata (a2) ----- */
/* Segments = maximal runs of equal consecutive ids in token order (reading R10): writes
   seg_start/seg_len/seg_id[0..n) and *n_seg_dev = n (all device int32 arrays of >= T entries).
   Bit-exact with the oracle's RLE.  The forwards do not consume it: they group tokens by adapter
   (route_kernel for T > 64, the decode kernels' group tables for T <= 64), which merges runs of the
   same id; this entry point exposes the SGMV segment view for callers (e.g. a scheduler) and tests. */
int bdlora_build_segments(const int32_t* ids, int64_t T, int32_t* seg_start, int32_t* seg_len,
                          int32_t* seg_id, int32_t* n_seg_dev, bdlora_stream_t stream);

/* ---------------------------------------------------------------- BD-LoRA forward ----------- */
/* Column layer, Alg. 2 lines 3-6 on device tp_rank -- NO communication:
     Y_i = X W_i + s_a (X A_i[a]) B_i[a]
   X  [T, d_in] bf16 (replicated input);  W = W_i^T as [M_loc, d_in] bf16 with the slices stacked
   (q_i | k_i | v_i rows);  ids [T] int32 device;  Y [T, M_loc] bf16 = [q_i | k_i | v_i] columns.
   Pool: COLUMN + BD.                                                                            */
int bdlora_column_forward(bdlora_pool* pool, const void* X, int64_t T, const void* W, const int32_t* ids,
                          void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);

/* Row layer partial, Alg. 1 lines 9-12 on device tp_rank, WITHOUT the all-reduce:
     P_i = X_i W_i + s_a (X_i A_i[a]) B_i[a]       (A_i = diagonal block, B_i = row shard)
   X [T, d_in/N] bf16;  W = W_i^T as [d_out, d_in/N] bf16;  P [T, d_out] bf16.  Pool: ROW + BD.   */
int bdlora_row_partial(bdlora_pool* pool, const void* X, int64_t T, const void* W, const int32_t* ids,
                       void* P, void* workspace, size_t ws_bytes, bdlora_stream_t stream);

/* Row layer, Alg. 1 lines 9-15: Y = AllReduce_i(P_i), the base model's own all-reduce -- the only
   collective of BD-LoRA.  Y [T, d_out] bf16, replicated; in-place NCCL bf16 sum.
   comm may be NULL iff tp_size == 1.                                                             */
int bdlora_row_forward(bdlora_pool* pool, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                       const int32_t* ids, void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);

/* Alg. 2 (a single column-parallel linear layer whose output is replicated): the column
   forward above on every device, then the base model's all-gather -- still no LoRA collective.
   Y [T, N * M_loc] bf16 = [Y_0 | Y_1 | ... | Y_{N-1}], the device blocks in rank order (for n_slices = 1
   exactly the full output X W + s X A B; for stacked slices the blocks keep their [q_i | k_i | v_i] order).
   T = 1: the device block is written straight into Y and gathered in place (the all-gather's rank-major
   layout IS [Y_0 | ... | Y_{N-1}]).  T > 1: the workspace (bdlora_workspace_bytes) holds the
   [N][T][M_loc] staging of the in-place ncclAllGather, interleaved into Y by one copy kernel.
   comm may be NULL iff tp_size == 1 (then it is bdlora_column_forward).  Pool: COLUMN + BD.          */
int bdlora_column_forward_gather(bdlora_pool* pool, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                                 const int32_t* ids, void* Y, void* workspace, size_t ws_bytes,
                                 bdlora_stream_t stream);

/* ---------------------------------------------------------------- S-LoRA comparison --------- */
/* Column: v_i = s X A[:, chunk i] -> ncclAllGather -> v [T, r] -> Y_i = X W_i + v B[:, cols i].
   Same tensors as bdlora_column_forward; pool COLUMN + SLORA.  +1 all-gather (merged over the
   J slices, P:340-341 footnote).                                                                 */
int slora_column_forward(bdlora_pool* pool, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                         const int32_t* ids, void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
/* Row (reading R12): v_i = s X_i A[rows i, :] -> ncclAllReduce -> v [T, r] ->
   P_i = X_i W_i, P_i[:, cols i] += v B[:, cols i] (the fused all-gather, zero extra traffic)
   -> base ncclAllReduce.  Pool ROW + SLORA.  +1 all-reduce.                                      */
int slora_row_forward(bdlora_pool* pool, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                      const int32_t* ids, void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);

/* ---------------------------------------------------------------- NFS-LoRA comparison ------- */
/* Column: every device holds the whole A_1, so v = s X A[a] (full rank, N-fold redundant)
   is local, and B_1[:, cols i] expands into the device's columns -- no communication.  Same tensors
   as bdlora_column_forward; pool COLUMN + NFS (no N | r requirement).                             */
int nfs_column_forward(bdlora_pool* pool, const void* X, int64_t T, const void* W, const int32_t* ids,
                       void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
/* Row: P_i = X_i W_i + s (X_i A[rows i, :]) B (B_2 whole on every device), then the base
   model's all-reduce -- the only collective, as for BD-LoRA.  comm may be NULL iff
   tp_size == 1; pool ROW + NFS.  nfs_row_partial is the same without the all-reduce.              */
int nfs_row_forward(bdlora_pool* pool, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                    const int32_t* ids, void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
int nfs_row_partial(bdlora_pool* pool, const void* X, int64_t T, const void* W, const int32_t* ids,
                    void* P, void* workspace, size_t ws_bytes, bdlora_stream_t stream);

/* ---------------------------------------------------------------- phases -------------------- */
/* The two device-local halves of every path, for callers that run the collective themselves
   (e.g. tests emulating N ranks on one GPU).  v is fp32 with layout [C][T][J][R_c]:
     R_c = max_rank/N (BD, S-LoRA column) or max_rank (S-LoRA row);  C = 1 except S-LoRA column
     after the all-gather, C = N (rank-major, chunk c = device c's shrink).
   bdlora_lora_shrink writes this device's [T][J][R_c] (C = 1):  v = s_a * X A_i[a]  (matmul_3/5).
   bdlora_base_expand computes Y = X W_i + expand(v) (matmul_1/2 + matmul_4/6 + add_1/2) reading v
   in the pool's post-collective layout (S-LoRA column: C = N).                                  */
int bdlora_lora_shrink(bdlora_pool* pool, const void* X, int64_t T, const int32_t* ids, float* v,
                       void* workspace, size_t ws_bytes, bdlora_stream_t stream);
int bdlora_base_expand(bdlora_pool* pool, const void* X, int64_t T, const void* W, const int32_t* ids,
                       const float* v, void* Y, void* workspace, size_t ws_bytes, bdlora_stream_t stream);
/* Elements of one device's v (= T * J * R_c) for this pool.                                      */
int bdlora_v_elems(const bdlora_pool* pool, int64_t T, int64_t* elems);

#ifdef __cplusplus
}
#endif
#endif /* BDLORA_H_ */
