/*
 * dscache.h -- C ABI of the B200 (sm_100a) DSCache streaming hot path.
 *
 * DSCache ("Decouple and Cache: KV Cache Construction for Streaming Video
 * Understanding", arxiv 2605.01858; text in PAPER.md) keeps, per stream and per
 * transformer layer, attention-sink K/V C_a, a FIFO cumulative
 * past cache U with budget l_U (Eq. 5-6), a feature buffer of
 * the newest l_I inputs (Eq. 3), builds an instant cache
 * I = phi(B, C_a) on demand (Eq. 7) and answers queries over
 * [C_a, U, I] (Eq. 8).  Keys are stored un-rotated
 * (position-agnostic encoding, Def. 4.1) and RoPE is applied
 * at use time with consecutive position ids from 0 over the active cache
 * (PAPER.md:236), so ids stay bounded on unbounded streams.
 *
 * One handle owns the device state of S independent streams x N layers x Hkv
 * KV heads (one GPU).  In the synthetic setting of this library the operator
 * phi of Eq. 4 is the caller's per-layer K/V: append_frame receives a frame's
 * raw K/V, the frame stays in the instant window for l_I steps, then becomes
 * part of the past window (reading Q2: disjoint windows in one ring).
 *
 * Conventions (all calls):
 *  - Tensor arguments are DEVICE pointers owned by the caller, dense row-major
 *    in the layouts stated per call; element type = config.dtype (bf16 or fp32).
 *    Base pointers must be 16-byte aligned.
 *  - Work is stream-ordered on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream).  No call synchronises the host except create,
 *    destroy, copy_ring, copy_sink.  Inputs may be reused once `stream` has
 *    passed the call.
 *  - Errors never cross the ABI as exceptions: every call returns a
 *    dscache_status; dscache_last_error() gives a thread-local message.
 *    Launch errors return DSCACHE_E_CUDA; asynchronous kernel faults surface at
 *    the caller's next synchronisation.
 *  - A handle is single-threaded (one host thread at a time).  Handles are
 *    independent (one per GPU / rank in multi-GPU runs).
 *  - All streams of a handle advance in lockstep (one frame per append per
 *    layer); layers may be advanced separately (layer_begin/layer_count), e.g.
 *    layer by layer as a real model produces them.
 */
#ifndef DSCACHE_H_
#define DSCACHE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dscache_s* dscache_t;   /* opaque; owns all device memory it allocates */

typedef enum {
  DSCACHE_OK = 0,
  DSCACHE_E_ARG = -1,           /* bad argument (null pointer, size, layer range, n_tokens)        */
  DSCACHE_E_CONFIG = -2,        /* invalid configuration at create                                  */
  DSCACHE_E_POS_OVERFLOW = -3,  /* A+W+max(C+q_max, tpf) > max_position (SPEC.md:112's overflow
                                   error, raised at create: re-based ids never exceed it afterwards) */
  DSCACHE_E_STATE = -4,         /* call out of order (attend before the sink, layers not in step)  */
  DSCACHE_E_CUDA = -5,          /* CUDA runtime error (launch / memcpy)                             */
  DSCACHE_E_OOM = -6            /* device allocation failed                                         */
} dscache_status;

enum { DSCACHE_DTYPE_BF16 = 0, DSCACHE_DTYPE_FP32 = 1 };
enum { DSCACHE_ROPE_SPLIT_HALF = 0,   /* pairs (i, i+d/2): Qwen2 / LLaVA-OV-7B (reading Q7, default) */
       DSCACHE_ROPE_ADJACENT = 1 };   /* pairs (2i, 2i+1)                                            */
enum { DSCACHE_INSTANT_RING = 0,     /* synthetic phi: a frame's K/V enter the ring on arrival and serve
                                        as its instant K/V for l_I steps, then as past (reading Q2)   */
       DSCACHE_INSTANT_EXTERNAL = 1 }; /* real-model mode: the instant segment's K/V
                                        are the caller's Eq. 7 output for this step; a frame enters
                                        the ring only when it leaves the buffer, with the K/V of its
                                        Eq. 5 update (dscache_append_past)                          */
enum { DSCACHE_IMPL_AUTO = 0,         /* tcgen05 kernel when eligible, else the SIMT kernel          */
       DSCACHE_IMPL_TC = 1,           /* force tcgen05 (E_CONFIG unless bf16, d=128, split-half RoPE)    */
       DSCACHE_IMPL_SIMT = 2 };       /* force the fp32 CUDA-core kernel                             */

typedef struct {
  int32_t num_streams;      /* S: independent video streams held by this handle                    */
  int32_t num_layers;       /* N: transformer layers                                               */
  int32_t num_q_heads;      /* Hq held by this handle (after any KV-head split)                    */
  int32_t num_kv_heads;     /* Hkv held by this handle; Hq % Hkv == 0; q head h reads kv head
                               h / (Hq/Hkv) (HF repeat_kv, reading Q10)                            */
  int32_t head_dim;         /* d in {64, 128}                                                      */
  int32_t kv_head_offset;   /* first global KV head of this handle (KV-head split); bookkeeping only */
  int32_t tokens_per_frame; /* tpf (196 for LLaVA-OV-7B)                             */
  int32_t sink_tokens;      /* A = l_A; 0 = no sink                                 */
  int32_t past_frames;      /* l_U: cumulative past budget in frames (W = l_U*tpf tokens)          */
  int32_t instant_frames;   /* l_I: feature-buffer / instant window in frames (C = l_I*tpf)        */
  int32_t max_query_tokens; /* q_max: largest n_q passed to attend                                 */
  int32_t max_position;     /* training length; create fails with E_POS_OVERFLOW if
                               A + W + max(C + q_max, tpf) > max_position (the largest id of the
                               attend and of the Eq. 5 update attention)                          */
  double  rope_theta;       /* RoPE base; theta_i = base^(-2i/d)                                   */
  int32_t rope_style;       /* DSCACHE_ROPE_*                                                      */
  int32_t dtype;            /* DSCACHE_DTYPE_*                                                     */
  int32_t device;           /* CUDA device ordinal the handle lives on                             */
  int32_t attn_impl;        /* DSCACHE_IMPL_*                                                      */
  int32_t instant_source;   /* DSCACHE_INSTANT_RING (default) or DSCACHE_INSTANT_EXTERNAL          */
} dscache_config;

typedef struct {
  int64_t frames_seen;         /* frames appended to this layer (sink excluded)                    */
  int64_t last_evicted_frame;  /* frame dropped from U at the latest append (Eq. 6), -1 if none    */
  int32_t sink_filled;         /* 1 once the A sink tokens are stored                              */
  int32_t past_tokens;         /* P_t = |U_t| in tokens                                            */
  int32_t instant_tokens;      /* C_t = |B_t| in tokens                                            */
  int32_t ring_slots;          /* R = W + C + tpf (one slack frame)                                */
  int32_t tail_slot;           /* ring slot of the oldest token of U (or of B when U is empty)     */
  int32_t instant_slot;        /* ring slot of the oldest instant token                            */
  int32_t max_key_id;          /* largest context key id of attend: A + P_t + C_t - 1              */
  int32_t max_query_id;        /* largest query id of attend with n_q = q_max                      */
  int32_t next_instant_tokens; /* C_{t+1}: instant tokens after the next frame (q_inst rows of the
                                  next dscache_step)                                                */
  int32_t instant_capacity;    /* C = l_I * tpf (the largest C_t)                                   */
} dscache_state;

/* Create a handle: validates the configuration, allocates the ring
 * [S][N][Hkv][R + 128][d] for K and V (raw, un-rotated; rows R..R+127 mirror slots
 * 0..127 so that any 128 consecutive slots are one contiguous box), the sink slabs [S][N][Hkv][A][d],
 * and the fp32 RoPE (cos, sin) table built in fp64 for ids 0 .. max_position-1.
 * The ring is zero-initialised (finite).  Synchronises the device.
 * Errors: E_ARG (null), E_CONFIG (d not in {64,128}, Hq % Hkv, budgets < 0, tpf < 1,
 * bf16 tcgen05 forced on an ineligible shape), E_POS_OVERFLOW, E_OOM, E_CUDA. */
dscache_status dscache_create(const dscache_config* cfg, dscache_t* out);

/* Release all device memory of the handle.  Synchronises the device. */
dscache_status dscache_destroy(dscache_t h);

/* Append one frame's raw K/V (or, on the first call of a layer when A > 0, the A
 * sink tokens) for layers [layer_begin, layer_begin+layer_count) of all S streams.
 *   k, v : [S][layer_count][n_tokens][Hkv][d]
 *   n_tokens: A on the first call of a layer with A > 0 (fills C_a, frozen afterwards,
 *             PAPER.md:113), tokens_per_frame afterwards; anything else -> E_ARG.
 * Frame f's token j goes to ring slot (f*tpf + j) mod R (contracted layout).  The
 * append realises Eq. 3 (push into the buffer window), Eq. 5 (the frame leaving
 * the buffer becomes past: a boundary move, no copy) and Eq. 6 (FIFO eviction of
 * frame t - l_I - l_U: a pointer move, zero bytes).  All layers of the range must
 * be at the same step (E_STATE otherwise). */
dscache_status dscache_append_frame(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                    const void* k, const void* v, int32_t n_tokens, void* stream);

/* Build the instant cache outputs (Eq. 7, I = phi(B, C_a)): every instant token i
 * (i < C_t, oldest first) attends to the sink and to instant tokens 0..i, never
 * to U (decoupled), with ids sink j -> j, instant i -> A + i
 * (PAPER.md:236); causal.  GQA flash attention with RoPE applied on load.
 *   q_inst : [S][layer_count][C_t][Hq][d]   (C_t from dscache_get_state)
 *   o_inst : [S][layer_count][C_t][Hq][d]   output, softmax(QK^T/sqrt(d)) V
 * C_t == 0 (l_I = 0) is a no-op.  E_STATE before the sink / first frame. */
dscache_status dscache_build_instant(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                     const void* q_inst, void* o_inst, void* stream);

/* Approximate instant cache: between the periodic full
 * rebuilds (dscache_build_instant, the "refresh"), only the newest frame's instant rows are
 * computed and the older rows are reused, so the per-step build costs O(C*tpf) instead of
 * O(C^2).  The rows are exactly the last tpf rows of dscache_build_instant at this step:
 * token j of frame t attends to the sink and to the instant window up to itself.
 *   q_new : [S][layer_count][tpf][Hq][d] ; o_new : [S][layer_count][tpf][Hq][d]
 * E_STATE before the sink and the first frame; E_CONFIG when l_I = 0. */
dscache_status dscache_build_instant_newest(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                            const void* q_new, void* o_new, void* stream);

/* The approximate instant cache as a library-driven state machine ("an extra
 * periodically refreshed cache for recent frames, enabling reuse of buffer-frame caches";
 * Table approx_cache periods 4/8/16; reading Q23).  The caller owns a persistent
 * row ring o_ring [S][layer_count][C][Hq][d], C = l_I*tpf: the rows of frame f live at ring
 * rows (f mod l_I)*tpf .. +tpf.  At step t (frame t the newest appended):
 *   refresh  (t mod period == 0, or the rows in o_ring are not this handle's rows of step t-1
 *            for the same period / o_ring / layer range): every buffer frame's rows are rebuilt
 *            as dscache_build_instant; q_rows holds the C_t instant queries oldest first;
 *   otherwise: only frame t's rows are built (as dscache_build_instant_newest, q_rows = its
 *            tpf queries); the rows of frames t-l_I+1..t-1 stay as built at their own step
 *            or at the last refresh.
 * So frame f's rows at step t are the Eq. 7 rows of step s_f = max(f, last refresh <= t):
 * context [sink | frames max(0, s_f-l_I+1) .. f], ids 0...  period = 1 is the
 * exact Eq. 7 build every step.  dscache_instant_approx_rows returns in *n_rows the query rows
 * the next dscache_build_instant_approx with these arguments takes (C_t or tpf); a mismatched
 * n_rows is E_ARG.  E_ARG for period < 1 or null pointers, E_CONFIG when l_I = 0 or in the
 * external-instant mode, E_STATE before the sink and the first frame. */
dscache_status dscache_instant_approx_rows(dscache_t h, int32_t layer_begin, int32_t layer_count, int32_t period,
                                           const void* o_ring, int32_t* n_rows);
dscache_status dscache_build_instant_approx(dscache_t h, int32_t layer_begin, int32_t layer_count, int32_t period,
                                            const void* q_rows, int32_t n_rows, void* o_ring, void* stream);

/* Fused all-gather epilogue of the KV-head split (P2): the attend
 * of this handle's KV heads (Eq. 8, as dscache_attend) with every output row stored by the
 * attention kernel itself to EACH of n_peers gathered-O buffers, instead of to a local O
 * followed by an all-gather.  peer_o[j] is a device pointer mapped in this process (a local
 * buffer, a P2P-enabled peer allocation, or a dscache_ipc_open mapping of another rank's
 * buffer), bf16 [S][layer_count][n_q][hq_total][d]; q head h of this handle lands at head
 * head_offset + h.  The stores are ordinary global stores on `stream`: the caller orders
 * them before any reader (stream sync + barrier, or an event).  Other arguments as
 * dscache_attend.  E_ARG unless 1 <= n_peers <= 8 with non-null pointers and
 * head_offset + Hq <= hq_total; E_CONFIG off the tcgen05 path. */
dscache_status dscache_attend_peers(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                    const void* q, const void* k_self, const void* v_self, int32_t n_q,
                                    void* const* peer_o, int32_t n_peers, int32_t hq_total, int32_t head_offset,
                                    void* stream);

/* CUDA IPC plumbing for dscache_attend_peers across processes of one node (NVLink /
 * NVSwitch): dscache_ipc_handle writes the 64-byte IPC handle of the device allocation
 * containing dev_ptr to handle_out and dev_ptr's byte offset inside it to *offset_out (a
 * caching allocator hands out interior pointers); dscache_ipc_open maps another process's
 * handle on `device` (lazy peer access enabled) and returns the allocation's base (add the
 * offset); dscache_ipc_close unmaps it.  E_CUDA on any CUDA error (e.g. opening a handle in
 * the process that exported it). */
dscache_status dscache_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
dscache_status dscache_ipc_open(int32_t device, const void* handle, void** dev_ptr_out);
dscache_status dscache_ipc_close(int32_t device, void* dev_ptr);

/* Resolution-boosted newest frame ("the buffer inputs may be temporarily
 * re-encoded, e.g. using a higher-resolution version of X_{t+1}, without modifying the
 * buffer itself"; PAPER.md:695 / Table "spa" PAPER.md:719-749).  The
 * instant cache is built from the buffer with its newest frame replaced by a caller-supplied
 * re-encoding of n_boost tokens (n_boost >= 1, any count: x1.5 / x2 spatial resolution gives
 * more tokens than tpf); the ring keeps the normal frame, so the cumulative update and every
 * later step are unchanged (reading Q22).  Keys [sink | older instant frames |
 * boosted frame], ids 0.. contiguous; query i at id A + i, causal.
 *   q_inst  : [S][layer_count][C_t - tpf + n_boost][Hq][d]  older instant tokens, then the
 *             boosted frame's tokens
 *   k_boost : [S][layer_count][n_boost][Hkv][d]   raw (un-rotated) K of the boosted frame
 *   v_boost : [S][layer_count][n_boost][Hkv][d]
 *   o_inst  : [S][layer_count][C_t - tpf + n_boost][Hq][d]
 * E_STATE before the sink and the first frame; E_CONFIG when l_I = 0; E_ARG for null
 * pointers or n_boost < 1; E_POS_OVERFLOW if A + C_t - tpf + n_boost > max_position. */
dscache_status dscache_build_instant_boost(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                           const void* q_inst, const void* k_boost, const void* v_boost,
                                           int32_t n_boost, void* o_inst, void* stream);

/* Attention of the query chunk over the final cache whose instant segment carries the
 * boosted newest frame: keys [sink | past | older instant frames | boosted frame (n_boost)
 * | self (n_q)], ids contiguous from 0, query i at
 * A + P_t + C_t - tpf + n_boost + i, causal inside the chunk (Eq. 8 with I built by
 * dscache_build_instant_boost).  Layouts as dscache_attend plus k_boost / v_boost as in
 * dscache_build_instant_boost.  The [boost | self] keys are gathered into a library-owned
 * scratch slab (device copies, stream-ordered) before the attention launch.
 * Errors as dscache_attend; E_ARG for n_boost < 1; E_CONFIG when l_I = 0. */
dscache_status dscache_attend_boost(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                    const void* q, const void* k_self, const void* v_self, int32_t n_q,
                                    const void* k_boost, const void* v_boost, int32_t n_boost, void* o,
                                    void* stream);

/* Real-model mode (config.instant_source = DSCACHE_INSTANT_EXTERNAL).
 * The instant cache I = phi(B, C_a) of Eq. 7 is new K/V for the buffer's
 * tokens built from a sink-only context, and the frame leaving the buffer gets yet another
 * K/V from the cumulative update phi(X_{t-l_I}, [C_a, zeta(U_{t-1})]) of Eq. 5
 * -- the same frame has different instant and past K/V.  In this mode:
 *
 * dscache_append_past: advances the layer range to step t (frame t arrived) and, once
 * t >= l_I, stores the Eq. 5 K/V of the frame leaving the buffer (frame t - l_I) into its
 * ring slots ((f*tpf + j) mod R, as the raw frames of the default mode); eviction and
 * position ids follow the same closed form (P_t, C_t).  k_past, v_past:
 * [S][layer_count][n_tokens][Hkv][d], n_tokens = tpf when t >= l_I, else 0 (pointers may be
 * NULL).  The first call of a layer with A > 0 must instead be dscache_append_frame with the
 * sink.  dscache_update_attend then runs the Eq. 5 attention of that frame over [sink |
 * zeta(U_{t-1}) | its own K/V just stored].  E_ARG for a wrong n_tokens, E_CONFIG in the
 * default mode. */
dscache_status dscache_append_past(dscache_t h, int32_t layer_begin, int32_t layer_count, const void* k_past,
                                   const void* v_past, int32_t n_tokens, void* stream);

/* Eq. 7 with the caller's instant K/V: the C_t instant tokens attend causally over
 * [sink | k_inst] with ids 0.., query i at A + i.
 *   q_inst, o_inst : [S][layer_count][C_t][Hq][d];  k_inst, v_inst : [S][layer_count][C_t][Hkv][d]
 * (raw, un-rotated).  E_CONFIG in the default mode, E_STATE before the sink and first step. */
dscache_status dscache_build_instant_ext(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                         const void* q_inst, const void* k_inst, const void* v_inst, void* o_inst,
                                         void* stream);

/* Eq. 8 with the caller's instant K/V: the query chunk over [sink | past (ring, P_t) | k_inst
 * (C_t) | self (n_q)], ids contiguous from 0, query i at A + P_t + C_t + i, causal inside the
 * chunk.  Layouts as dscache_attend plus k_inst / v_inst as dscache_build_instant_ext; the
 * [instant | self] keys are gathered into per-call stream-ordered scratch.  E_CONFIG in the
 * default mode; otherwise errors as dscache_attend. */
dscache_status dscache_attend_ext(dscache_t h, int32_t layer_begin, int32_t layer_count, const void* q,
                                  const void* k_self, const void* v_self, int32_t n_q, const void* k_inst,
                                  const void* v_inst, void* o, void* stream);

/* Decoding in the real-model mode (PAPER.md:128 over C_{t+1} = [C_a, U, I], Q25): the last
 * n_q tokens of an n_self-token self segment (the query chunk and the tokens generated so
 * far) attend over [sink | past (ring, P_t) | k_inst (C_t) | self], ids contiguous from 0,
 * causal inside self.  k_inst / v_inst are the step's instant K/V as for dscache_attend_ext;
 * q [S][lc][n_q][Hq][d], k_self / v_self [S][lc][n_self][Hkv][d], o like q.  E_ARG unless
 * 1 <= n_q <= n_self; E_CONFIG in the default mode; other errors as dscache_decode. */
dscache_status dscache_decode_ext(dscache_t h, int32_t layer_begin, int32_t layer_count, const void* q,
                                  const void* k_self, const void* v_self, int32_t n_self, int32_t n_q,
                                  const void* k_inst, const void* v_inst, void* o, void* stream);

/* Attention of an n_q-token query chunk over [C_a | U | I | self] (Eq. 8 plus the
 * chunk's own K/V, which are used and then discarded: PAPER.md:212/699).  Ids:
 * sink 0..A-1, past+instant A..A+P_t+C_t-1 (oldest first), query/self token i at
 * A+P_t+C_t+i (Eq. 2's l_A+l_W once the window is full); causal inside the chunk.
 *   q      : [S][layer_count][n_q][Hq][d]
 *   k_self : [S][layer_count][n_q][Hkv][d]   raw (un-rotated) K of the chunk
 *   v_self : [S][layer_count][n_q][Hkv][d]
 *   o      : [S][layer_count][n_q][Hq][d]    output
 * 1 <= n_q <= max_query_tokens, else E_ARG.  E_STATE before the first frame. */
dscache_status dscache_attend(dscache_t h, int32_t layer_begin, int32_t layer_count,
                              const void* q, const void* k_self, const void* v_self, int32_t n_q,
                              void* o, void* stream);

/* Decoding: "autoregressive decoding is performed using
 * the KV cache C_{t+1}".  The last n_q tokens of a transient self segment of n_self >= n_q
 * tokens (the query chunk followed by the tokens generated so far; their K/V are used and
 * discarded) attend over [sink | past | instant | self], causal inside
 * self; self token j has id A + P_t + C_t + j.  n_q = 1 is one decode step.
 *   q      : [S][layer_count][n_q][Hq][d]       queries of the last n_q self tokens
 *   k_self : [S][layer_count][n_self][Hkv][d]   raw K of the self segment
 *   v_self : [S][layer_count][n_self][Hkv][d]
 *   o      : [S][layer_count][n_q][Hq][d]
 * E_ARG unless 1 <= n_q <= n_self; E_POS_OVERFLOW if A + P_t + C_t + n_self > max_position. */
dscache_status dscache_decode(dscache_t h, int32_t layer_begin, int32_t layer_count,
                              const void* q, const void* k_self, const void* v_self, int32_t n_self,
                              int32_t n_q, void* o, void* stream);

/* Decoding over a sampled cumulative cache (zeta_decode: "we also sample the
 * cumulative KV cache at 0.5 FPS during decoding"; reading Q24): as dscache_decode,
 * but the past segment keeps only every past_stride-th frame of U, anchored at its newest
 * frame (frames j = n_past-1, n_past-1-stride, ... >= 0, oldest first); the kept keys get
 * contiguous ids: sink 0..A-1, kept past A.., instant, then self.
 * past_stride = 1 is dscache_decode.  The memory-bound decode kernel serves bf16, d = 128,
 * split-half RoPE and n_q * Hq/Hkv <= 16 (one 16-row tile per kv head, all q heads of the
 * group sharing every K/V byte read); other decodes run through the attention kernel, or
 * with past_stride > 1 through the SIMT kernel.  E_ARG for past_stride < 1; other errors
 * as dscache_decode. */
dscache_status dscache_decode_sampled(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                      const void* q, const void* k_self, const void* v_self, int32_t n_self,
                                      int32_t n_q, int32_t past_stride, void* o, void* stream);

/* Cumulative-update attention of Eq. 5: at step t
 * the input X_{t-l_I} that just left the buffer is encoded as phi(X_{t-l_I},
 * [C_a, zeta(U_{t-1})]); this call runs its attention: each of the tpf tokens of frame
 * e = t - l_I attends to the sink, to zeta(U_{t-1}) = the newest active_frames frames
 * of the cumulative cache before the update (l_L <= l_U; active_frames
 * is clamped to the frames U_{t-1} holds), and to the tokens of frame e up to itself.
 * Ids are consecutive from 0 over that active cache.  The keys are the
 * raw K/V already in the ring: frames e-l_L .. e are contiguous there (the one slack
 * frame of the ring keeps the frame Eq. 6 evicts at step t readable during step t).
 *   q_upd : [S][layer_count][tpf][Hq][d]   queries of frame e's tokens
 *   o_upd : [S][layer_count][tpf][Hq][d]   output
 * E_STATE before step l_I (nothing has left the buffer), E_ARG if active_frames < 0. */
dscache_status dscache_update_attend(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                     const void* q_upd, void* o_upd, int32_t active_frames, void* stream);

/* One streaming step of the hot path for a layer range:
 * exactly dscache_append_frame(k_frame, v_frame, tpf) + dscache_build_instant(q_inst,
 * o_inst) + dscache_attend(q, k_self, v_self, n_q, o), with identical results.  When both
 * attention calls take the tcgen05 kernel (and no debug capture is set) the build and the
 * attend run as ONE persistent launch: attend items first (longest), build items after,
 * so the SMs the attend leaves idle at its tail run the build (Eq. 3 + Eq. 7 + Eq. 8).
 * Arguments and layouts as in the three calls; all device pointers, stream-ordered.
 * Errors as the three calls; E_STATE before the sink was appended. */
dscache_status dscache_step(dscache_t h, int32_t layer_begin, int32_t layer_count,
                            const void* k_frame, const void* v_frame, const void* q_inst, void* o_inst,
                            const void* q, const void* k_self, const void* v_self, int32_t n_q, void* o,
                            void* stream);

/* Context-parallel building blocks: the attend of dscache_attend split
 * over its keys.  The keys of every (stream, layer, kv head, m-block) work item -- sink and
 * self rows, then the [past | instant] window in 64-key tiles, all with their full-context
 * ids -- are cut into n_parts contiguous tile ranges; this call computes
 * range `part` only and writes the partial softmax attention over it:
 *   o_part   : DEVICE fp32 [S][layer_count][n_q][Hq][d], O_part = sum_j p_j v_j / sum_j p_j
 *   lse_part : DEVICE fp32 [S][layer_count][n_q][Hq], log2 of sum_j 2^(s_j log2e / sqrt(d))
 * Softmax attention is invariant to how the key set is split, so combining the n_parts
 * partials (dscache_combine_partials, on any rank after an all-gather) equals
 * dscache_attend up to rounding.  tcgen05 path only (E_CONFIG otherwise); E_ARG if a part
 * would get no keys or n_q is out of range. */
dscache_status dscache_attend_partial(dscache_t h, int32_t layer_begin, int32_t layer_count,
                                      const void* q, const void* k_self, const void* v_self, int32_t n_q,
                                      int32_t part, int32_t n_parts, float* o_part, float* lse_part,
                                      void* stream);
/* O = sum_r 2^(lse_r - M) O_r / sum_r 2^(lse_r - M), M = max_r lse_r (partials with
 * lse = -inf weigh 0).  o_parts: DEVICE fp32 [n_parts][rows][d], lse_parts: [n_parts][rows],
 * o: DEVICE bf16 [rows][d] (rows = S*layer_count*n_q*Hq for attend partials). */
dscache_status dscache_combine_partials(dscache_t h, int32_t n_parts, int64_t rows, const float* o_parts,
                                        const float* lse_parts, void* o, void* stream);

/* Host counters of `layer` (closed form of Eq. 3/5/6 at the latest append). */
dscache_status dscache_get_state(dscache_t h, int32_t layer, dscache_state* out);

/* Test/checkpoint: synchronous copy of the ring of (stream, layer) to HOST memory,
 * slot-exact, each [Hkv][R][d] in the config dtype. */
dscache_status dscache_copy_ring(dscache_t h, int32_t stream_idx, int32_t layer,
                                 void* k_host, void* v_host);

/* Test/checkpoint: synchronous copy of the sink slab of (stream, layer), [Hkv][A][d]. */
dscache_status dscache_copy_sink(dscache_t h, int32_t stream_idx, int32_t layer,
                                 void* k_host, void* v_host);

/* Checkpoint restore (SURVEY §5 checkpoint / resume; "bit-exact round trip").
 * The streaming state of a handle is the host counters of each layer plus the device ring and
 * sink slabs (everything later steps read is U, A and the frame counter).
 * A checkpoint is dscache_get_state + dscache_copy_ring + dscache_copy_sink for every
 * (stream, layer); a handle created with the same config and given these three calls resumes
 * with results bit-identical to the uninterrupted handle's (same kernels, same inputs).
 * restore_ring : HOST [Hkv][R][d] each, the layout dscache_copy_ring writes; also refreshes the
 *                mirror rows R..R+127 (create's layout).  Synchronous: waits for the device
 *                before and after, so no queued kernel reads half-replaced rows.
 * restore_sink : HOST [Hkv][A][d] each (no-op when A = 0).  Synchronous.
 * set_state    : the counters of `layer`: frames_seen (>= 0) and sink_filled (0/1) as
 *                dscache_get_state reported them; the last evicted frame follows from the
 *                closed form (Eq. 6).  The approximate instant cache (NEXT-3) restarts its
 *                reuse chain: the next dscache_build_instant_approx refreshes (exact rows).
 * Errors: E_ARG (null, out of range), E_STATE (frames without a sink, sink_filled = 0 when
 * A = 0), E_CUDA. */
dscache_status dscache_restore_ring(dscache_t h, int32_t stream_idx, int32_t layer,
                                    const void* k_host, const void* v_host);
dscache_status dscache_restore_sink(dscache_t h, int32_t stream_idx, int32_t layer,
                                    const void* k_host, const void* v_host);
dscache_status dscache_set_state(dscache_t h, int32_t layer, int64_t frames_seen, int32_t sink_filled);

/* Debug exports (K7).  build_pos / attend_pos: NULL = off, else DEVICE int32
 * buffers of num_streams * num_layers * dscache_debug_len(h) entries, one block of
 * dscache_debug_len(h) per (stream, layer) ([S][N][len], int32), which the attention and
 * staging kernels fill, for kv head 0 of every (stream, layer) of a call (fused
 * dscache_step and staged builds included), with the position ids they actually applied: [0,A) sink keys, [A,A+R) ring slot -> id (untouched if the
 * slot is not in the window), [A+R, A+R+M) self keys, [A+R+M, A+R+2M) queries,
 * M = max(C, q_max).  poison != 0: after each append the slots of the frame just
 * evicted are overwritten with a large finite sentinel (finite, not NaN). */
dscache_status dscache_set_debug(dscache_t h, int32_t* build_pos, int32_t* attend_pos, int32_t poison);
int32_t        dscache_debug_len(dscache_t h);

/* Per-CTA event timeline of the tcgen05 attention kernel (profiling aid).  Recorded only
 * by a library built with -DFA_TRACE=1 (scripts/trace_fa.py builds that variant and prints
 * the timeline); the production library accepts the call and records nothing.  buf: DEVICE
 * int64 buffer of ntrace_cta * 32 * 1024 entries (NULL = off): for the first ntrace_cta CTAs
 * of each launch, clock64() at [cta][event][index] for the 32 events of attn_fa.cu (FT_*:
 * per tile, the MMA issuers' waits for P0 / P1 / K / V and their S / PV issue, S seen and P
 * written by each softmax warpgroup, K landed and rotated, the copy warps' issues, the
 * softmax phases of warp 0; per item, item start, Q tiles ready, O read out, epilogue and
 * Q-prep boundaries; the CTA end).  Indices >= 1024 are not recorded. */
dscache_status dscache_set_trace(dscache_t h, int64_t* buf, int32_t ntrace_cta);

/* Profiling: when enabled, every attention/combine kernel launch is bracketed by
 * CUDA events on the caller's stream; read accumulates the device time (ms) and
 * launch counts since the last reset, per kind (0 = build_instant, 1 = attend).
 * kernel_launches counts every kernel this handle launched (append, attention,
 * combine).  read synchronises the events it consumes. */
dscache_status dscache_profile(dscache_t h, int32_t enable);
dscache_status dscache_profile_read(dscache_t h, double* ms_build, double* ms_attend,
                                    int64_t* n_build, int64_t* n_attend, int64_t* kernel_launches,
                                    int32_t reset);

/* Which attention kernel serves build_instant (which=0) / attend (which=1) on this
 * handle: DSCACHE_IMPL_TC or DSCACHE_IMPL_SIMT. */
int32_t dscache_attn_impl(dscache_t h, int32_t which);

/* Debug: pipeline-watchdog records of the tcgen05 kernel.  With the environment variable
 * DSC_WATCHDOG=1 set before the first launch, a kernel wait that spins ~2^31 cycles writes
 * (cta, warp, barrier index, parity, clock) into host-mapped memory before trapping; this
 * copies n uint64 words of that record (word 0 = number of records, then 4 words each) to
 * out.  The memory is host memory, so it stays readable after the context has died.
 * Returns 0, or -1 when the watchdog record is not enabled. */
int32_t dscache_watchdog_read(uint64_t* out, int32_t n);

/* Thread-local message of the last failing call ("" if none). */
const char* dscache_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DSCACHE_H_ */
