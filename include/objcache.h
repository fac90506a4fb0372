/*
 * objcache.h -- C ABI of the B200-native ObjectCache hot path (arxiv 2605.22850).
 *
 * The library assembles a prefix-cache hit the way ObjectCache's storage server
 * does (Sec. 3.3; Alg. A1): a request names
 * N hash-addressed KV chunks, each stored chunk-major (KV_L2TD), and
 * for every layer l the library moves byte range [lS, (l+1)S) of every chunk,
 * in prefix order, into the caller's GPU KV memory, announcing each layer as
 * soon as it is complete so prefill of layer l overlaps the transfer of l+1
 * (Sec. 3.5, Eq. 3).  On B200 the "storage server" is a CUDA kernel
 * reading an HBM, pinned-host or peer-GPU chunk store; the "RDMA target" is the
 * serving engine's paged KV cache (or the paper's flat client buffer); the
 * layer-ready notification is a device counter / CUDA event per layer.
 *
 * Conventions for every entry point:
 *  - Return value: OC_OK (0) or a negative OC_E* code; the thread-local text of
 *    the last failure is in oc_last_error().  No entry point aborts the process.
 *  - "device address" = a CUDA UVA address the store's GPU can dereference: its
 *    own HBM, mapped pinned host memory, or a peer GPU's memory with peer access.
 *  - Streams are cudaStream_t passed as void* (NULL = the legacy default stream).
 *  - Host arrays passed in are read during the call only (copied if kept).
 *  - Objects (oc_store, oc_desc) are owned by the library and freed by the
 *    matching *_destroy / *_free call.  KV destination memory and streams are
 *    owned by the caller.
 *
 * No CPU fallback exists: every byte of the data path is moved by the library's
 * sm_100a kernels; without a usable GPU the data-path calls return OC_ECUDA.
 */
#ifndef OBJCACHE_H
#define OBJCACHE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define OC_API __attribute__((visibility("default")))
#else
#define OC_API
#endif

#define OC_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------- */
#define OC_OK 0
#define OC_EINVAL (-1)      /* bad argument or inconsistent layout               */
#define OC_ENOMEM (-2)      /* host or device allocation failed                  */
#define OC_ENOTFOUND (-3)   /* a chunk key is not in the store (see bad_index)   */
#define OC_EIMMUTABLE (-4)  /* put of an existing key with different bytes       */
#define OC_ERANGE (-5)      /* index/size out of range (layer >= L, small target)*/
#define OC_EALIGN (-6)      /* address or stride not a multiple of 16 bytes      */
#define OC_ECUDA (-7)       /* CUDA runtime/driver error (text in oc_last_error) */
#define OC_EFULL (-8)       /* store capacity exhausted                          */
#define OC_ENOTSUP (-9)     /* option not supported in this configuration        */

/* ---- geometry ----------------------------------------------------------- */
/* A rolling-hash chunk key H_i = SHA-256(H_{i-1} || LE-u32 tokens_i), root = 32
 * zero bytes (the paper names only "Hash", reading c1). */
typedef struct { uint8_t b[32]; } oc_key;

/* Eq. 1 symbols: L layers, n_kv KV heads, head dim d, element width
 * p bytes, G tokens per chunk.  Derived: row = n_kv*d*p (one token of K or V at
 * one layer), S = 2*G*row (one layer of one chunk), chunk object = L*S bytes,
 * laid out [L][2 (K,V)][G][n_kv][d] (KV_L2TD, reading c2). */
typedef struct {
    uint32_t num_layers;
    uint32_t kv_heads;
    uint32_t head_dim;
    uint32_t elem_bytes;
    uint32_t chunk_tokens;
} oc_layout;

/* Fills row bytes, S and L*S.  EINVAL if a field is 0 or L*S overflows. */
OC_API int oc_geometry(const oc_layout* layout, uint64_t* row_bytes, uint64_t* layer_chunk_bytes,
                       uint64_t* chunk_bytes);

/* Slot pitch: the byte distance between consecutive chunk slots of a store slab
 * of this layout and tier (slot i at slab base + i*pitch; an object's L*S bytes
 * at the start of its slot).  The layout of a slot is the paper's chunk object
 * (P:347-354); how slots are spaced is this library's choice: an HBM slab of
 * chunks of >= 1 MiB spaces them by the smallest multiple of 32 KiB >= L*S whose
 * count of 32 KiB granules has no factor 3, 5 or 7 (a layer reads one S-byte slice
 * per slot, and on B200 such spacings read up to 9% faster than e.g. 2.5 or 5 MiB;
 * profiles/r02_pitch_sweep.txt); pinned-host slabs and smaller chunks are
 * dense (pitch = L*S).  Pure function (no GPU).  EINVAL on a bad layout, tier or
 * null out. */
OC_API int oc_slot_pitch(const oc_layout* layout, int tier, uint64_t* pitch);

/* Eq. 2: returns OC_DELIVER_CHUNK_MAJOR if W < theta, else
 * OC_DELIVER_LAYER_MAJOR (theta = 0 always selects layer-major). */
OC_API int oc_select_mode(uint64_t payload_W, uint64_t theta);

/* ---- keys (host) -------------------------------------------------------- */
/* SHA-256 (FIPS 180-4) of n bytes. */
OC_API int oc_sha256(const void* data, uint64_t n, uint8_t out[32]);

/* Keys of the floor(n_tokens/G) complete G-token blocks of `tokens`, chained
 * from `parent` (NULL = root).  Writes min(count, cap) keys, sets *n_out = count.
 * A trailing partial block is ignored.  ERANGE if cap < count. */
OC_API int oc_chunk_keys(const uint32_t* tokens, uint64_t n_tokens, uint32_t chunk_tokens,
                         const oc_key* parent, oc_key* out, uint64_t cap, uint64_t* n_out);

/* chunk_keys_batch: the same keys computed on the GPU for a batch of token streams (the offload
 * path's keys).  Request r's tokens are tokens[tok_off[r] .. + n_tokens[r]),
 * its floor(n_tokens[r]/G) keys are written to out[key_off[r] ..], chained from parents[r]
 * (parents NULL = the root for every request).  tokens, tok_off, n_tokens, parents, out and
 * key_off are DEVICE arrays of the current device; the caller sizes them (no bounds are checked).
 * One thread per request (a chain is sequential): a single chain is slower than oc_chunk_keys on
 * the host, a batch of hundreds of requests is much faster.  Asynchronous on `stream`. */
OC_API int oc_chunk_keys_batch(const uint32_t* tokens, const uint64_t* tok_off, const uint64_t* n_tokens,
                               uint32_t n_requests, uint32_t chunk_tokens, const oc_key* parents, oc_key* out,
                               const uint64_t* key_off, void* stream);

/* ---- chunk store -------------------------------------------------------- */
typedef enum { OC_TIER_HBM = 0, OC_TIER_PINNED_HOST = 1 } oc_tier;
typedef struct oc_store oc_store;

/* Create a store of `capacity_chunks` slots of L*S bytes on GPU `device`:
 * HBM (cudaMalloc) or pinned, mapped host memory (cudaHostAlloc; the GPU reads
 * it over PCIe -- the stand-in for the paper's RDMA landing zone). */
OC_API int oc_store_create(const oc_layout* layout, int tier, int device, uint64_t capacity_chunks,
                           oc_store** out);
OC_API int oc_store_destroy(oc_store* store);
OC_API int oc_store_count(const oc_store* store, uint64_t* n_chunks);
/* Hot layers (pinned-host stores, before the first put): mirror the first `hot_layers` layers of
 * every chunk in HBM (hot_layers*S bytes per slot, cudaMalloc'd now).  A fetch whose chunks all
 * carry the mirror reads those layers from HBM with a full grid -- its exposed first-layer
 * latency X0 drops from one layer over PCIe to one layer at HBM speed -- and the
 * rest from host memory.  EINVAL: HBM or imported store, or chunks already stored; ERANGE:
 * hot_layers > L.  put_from_paged into such a store is ENOTSUP. */
OC_API int oc_store_set_hot_layers(oc_store* store, uint32_t hot_layers);

/* The mirror depth that hides the host link (Eq. 3): with X seconds per layer over the
 * link and C seconds of compute per layer, the smallest K >= 1 such that mirroring layers < K lets
 * the free-running pipeline add no TTFT: K = max(1, ceil(L - (L-1) C / X)), clamped to L.  Pure.
 * EINVAL if X or C is not finite and > 0, or L = 0. */
OC_API int oc_hot_layers_for(double X_s, double C_s, uint32_t L, uint32_t* K);

/* Slab base device address and size in bytes = capacity * oc_slot_pitch (for
 * IPC export and tests). */
OC_API int oc_store_slab(const oc_store* store, uint64_t* base, uint64_t* bytes);

/* put_chunks (P:224 offload; P:36-40 immutable, content-addressed writes):
 * store n chunk objects; payloads = n*L*S contiguous bytes, host or device
 * memory.  An existing key with identical bytes is deduplicated; with
 * different bytes the call fails with EIMMUTABLE and *bad_index = its index
 * (chunks before it are stored).  *n_new = number of keys that were new.
 * EFULL when capacity is exhausted.  Thread-safe.  Device payloads are read
 * after all work enqueued so far on the legacy default stream (and on streams
 * that synchronize with it); a producer on a non-blocking stream must be
 * synchronized by the caller first.  Returns when the bytes are stored. */
OC_API int oc_put_chunks(oc_store* store, const oc_key* keys, const void* payloads, uint64_t n,
                         uint64_t* n_new, uint64_t* bad_index);

/* match_prefix: hash the complete G-blocks of `tokens`
 * from `parent` (NULL = root) and return the longest leading run of keys
 * present in the store, in prefix order (reading c17).  Writes up to `cap`
 * keys; *n_matched = run length (ERANGE if it exceeds cap). */
OC_API int oc_match_prefix(oc_store* store, const uint32_t* tokens, uint64_t n_tokens,
                           const oc_key* parent, oc_key* out, uint64_t cap, uint64_t* n_matched);

/* Resolve keys to the device addresses of their slots.  ENOTFOUND with
 * *bad_index = first missing key. */
OC_API int oc_store_lookup(oc_store* store, const oc_key* keys, uint64_t n, uint64_t* addrs,
                           uint64_t* bad_index);

/* Make `peer`'s chunks resolvable through `store` (peer keys are looked up
 * after local ones).  `peer` must outlive `store`'s descriptors, and its slab
 * must be readable from `store`'s GPU (same GPU, peer access, or host tier).
 * OC_EINVAL if the attachment would close a cycle (peer already reaches store). */
OC_API int oc_store_attach_peer(oc_store* store, oc_store* peer);

/* Multi-process sharing of an HBM store (config 5, NVLink P2P):
 * export writes an opaque blob (CUDA IPC handle + key table) of *size bytes
 * (call with buf = NULL to query the size); import opens it in another process
 * as a read-only peer store bound to GPU `device`, usable with attach_peer.  The blob
 * carries the exporter's slot pitch.  import: EINVAL for a blob that is not an
 * export of this library version, is truncated, names slots beyond its capacity,
 * or whose capacity x pitch exceeds the mapped allocation. */
OC_API int oc_store_export(oc_store* store, void* buf, uint64_t* size);
OC_API int oc_store_import(const void* buf, uint64_t size, int device, oc_store** out);

/* ---- descriptor (Table 1) ------------------------------------ */
typedef enum { OC_DELIVER_LAYER_MAJOR = 0, OC_DELIVER_CHUNK_MAJOR = 1 } oc_delivery;
typedef enum { OC_TARGET_PAGED = 0, OC_TARGET_FLAT = 1 } oc_target_kind;

/* The descriptor's rdma_target, made GPU-native (reading c4).
 * PAGED: request token u (u = first_token + j*G + t for token t of chunk j),
 *   matrix K or V, head h, at layer l is written to
 *     {k,v}_base[l] + block_table[u / block_size]*block_stride
 *                   + (u % block_size)*token_stride + h*head_stride
 *   as d*p bytes.  NHD (vLLM FlashAttention): token_stride = row,
 *   head_stride = d*p.  HND: token_stride = d*p, head_stride = block_size*d*p.
 *   block_table[0 .. num_blocks) covers tokens [0, num_blocks*block_size);
 *   the blocks used must be distinct and >= 0.  Slots outside the prefix are
 *   not touched (reading c5).
 * FLAT: the paper's client_buffer (Alg. A1 line 6): layer l's payload B_l of
 *   N*S bytes at flat_base + l*N*S, chunk j at offset j*S; needs
 *   flat_capacity >= N*L*S.
 * Every base address, stride and d*p must be a multiple of 16 (EALIGN). */
typedef struct {
    uint32_t kind;
    uint32_t block_size;
    uint32_t first_token;
    uint32_t reserved;
    const uint64_t* k_base;      /* host array [L] of device addresses */
    const uint64_t* v_base;      /* host array [L] of device addresses */
    uint64_t block_stride;
    uint64_t token_stride;
    uint64_t head_stride;
    const int32_t* block_table;  /* host array [num_blocks] */
    uint64_t num_blocks;
    uint64_t flat_base;          /* device address */
    uint64_t flat_capacity;      /* bytes */
} oc_target;

typedef struct oc_desc oc_desc;

/* build_descriptor: validate the request and resolve every key to its chunk
 * slot (local store first, then attached peers), then upload the packed
 * device descriptor {src[N], block table, K/V bases} with one H2D copy.
 * Errors: EINVAL (n = 0, layout != store layout, duplicate/negative block ids,
 * unknown kind), ENOTFOUND (*bad_index = first missing key in prefix order),
 * ERANGE (target too small), EALIGN. */
OC_API int oc_build_descriptor(oc_store* store, const oc_key* keys, uint64_t n, const oc_layout* layout,
                               int delivery, const oc_target* target, oc_desc** out,
                               uint64_t* bad_index);
OC_API int oc_desc_free(oc_desc* desc);
/* N, W = N*L*S, and the number of copy units per layer. */
OC_API int oc_desc_info(const oc_desc* desc, uint64_t* n_chunks, uint64_t* payload_W,
                        uint64_t* units_per_layer);

/* put_from_paged -- the offload path ("newly produced KV blocks are offloaded back to
 * object storage for future reuse"): chunk j of a request (its tokens first_token + j*G ..
 * + G-1) is gathered from the paged KV cache described by `target` (OC_TARGET_PAGED, same address
 * rule as build_descriptor) into a new slot in KV_L2TD order, on `stream` (asynchronous: later
 * fetches of these keys must be ordered after `stream`).  Keys already in the store are
 * deduplicated without reading their bytes (identity is the prefix-chain key, reading c18).
 * *n_new = new keys.  Errors as build_descriptor, plus EFULL (*bad_index = first key that did
 * not fit; earlier new keys are stored). */
OC_API int oc_put_from_paged(oc_store* store, const oc_key* keys, uint64_t n, const oc_layout* layout,
                             const oc_target* target, void* stream, uint64_t* n_new, uint64_t* bad_index);

/* ---- fetch (Alg. A1 on the GPU) ------------------------------------------ */
typedef enum {
    OC_FETCH_PERSISTENT = 0, /* one launch covers all layers; per-layer device
                                counters; wait_layer = stream wait-value      */
    OC_FETCH_PER_LAYER = 1,  /* one launch + one CUDA event per layer         */
} oc_fetch_mode;

typedef enum {
    OC_COPY_LDST = 0,        /* 16-byte vector loads/stores through registers */
    OC_COPY_BULK = 1,        /* TMA bulk copies through a shared-memory ring  */
    OC_COPY_CE = 2,          /* pinned-host chunks only (ENOTSUP otherwise): per layer, one
                                strided copy-engine transfer per run of consecutive store slots
                                into a double-buffered HBM stage (2*N*S bytes, owned by the
                                descriptor), then the BULK kernel scatters the stage into the
                                target and announces the layer.  PERSISTENT mode, unpaced.
                                With a FLAT target the copies land in the client buffer
                                directly (no stage, no scatter kernel).
                                ~55 GB/s of PCIe reads vs ~51 for SM zero-copy; the saturated
                                PCIe queue adds ~5 us to each launch of other streams.       */
    OC_COPY_AUTO = 3,        /* CE for an unpaced PERSISTENT fetch into a FLAT target
                                from pinned-host chunks in at most 4 slot runs;
                                else BULK when destination rows are contiguous
                                (NHD, flat target) or strict pacing is asked
                                for, else LDST (head-split targets such as
                                HND); the default                               */
} oc_copy_engine;

typedef struct {
    uint32_t mode;           /* oc_fetch_mode                                   */
    uint32_t engine;         /* oc_copy_engine                                  */
    uint32_t max_ctas;       /* copy-CTA cap (SM budget when co-running); 0 = auto:
                                the whole GPU for HBM sources, 8 CTAs when most
                                chunks live in pinned host memory (PCIe-bound:
                                enough for the link, a short read queue)         */
    uint32_t unit_bytes;     /* bytes per work unit (a run of rows of one chunk's
                                layer slice); 0 = auto: 32 KiB, or 64 KiB when an
                                HBM-sourced fetch has a budget of <= 1 CTA/SM    */
    double pace_Bps;         /* minimal pacer: layer l is released no
                                earlier than t0 + l*(N*S)/pace_Bps; 0 = off.
                                PERSISTENT mode only.                           */
    uint32_t pace_strict;    /* 1: byte-granular pacing instead -- byte b of the
                                fetch (layer-major) is released no earlier than
                                t0 + b/pace_Bps, so the request never exceeds its
                                rate (the held rate of Alg. A2 line 6)          */
    uint32_t flags;          /* OC_FETCH_OVERLAP: the launch may start while the
                                stream's previous fetch launch is still draining
                                (programmatic dependent launch, no wait on its
                                memory): the caller guarantees the work before it
                                on the stream neither writes this fetch's
                                destination nor produces anything it reads (e.g.
                                back-to-back fetches of different requests).  The
                                previous fetch's tail and this one's ramp overlap.
                                Single-descriptor kernel launches (BULK, LDST);
                                the CE engine and batches ignore it.  0 = stream
                                order.                                           */
} oc_fetch_opts;
#define OC_FETCH_OVERLAP 1u
/* OC_FETCH_FIRST_LAYER_FULL: with max_ctas set, layer 0 (the exposed X_0 of Eq. 3,
 * P:457-460) is copied by the whole GPU and only layers 1..L-1 by max_ctas CTAs --
 * for a fetch co-running with prefill compute, which needs layer 0 at once and
 * the rest at the compute's pace (two launches; each announces its layers).
 * PERSISTENT mode, kernel engines. */
#define OC_FETCH_FIRST_LAYER_FULL 2u
/* OC_FETCH_YIELD: layer 0 with the whole GPU as a persistent launch, then layers
 * 1..L-1 with one work unit per CTA (a grid of all their units): CTAs retire as they
 * finish, so the kernels of a higher-priority stream (the co-running prefill) take
 * their SMs as soon as they are launched and the fetch fills the rest.  Use with a
 * low-priority copy stream.  PERSISTENT mode, BULK engine, HBM-resident chunks. */
#define OC_FETCH_YIELD 4u

/* OC_FETCH_LEAN: the TMA engine's copy CTAs keep the smallest shared-memory ring
 * (two units), so with small units (unit_bytes = 8192: ~18 KiB per CTA) a copy CTA
 * fits on an SM beside a co-running GEMM's CTA (cuBLAS sm_100 tiles leave ~19 KiB)
 * instead of excluding it.  PERSISTENT mode, BULK engine. */
#define OC_FETCH_LEAN 16u

/* fetch_layerwise: enqueue the transfer of all L layers on `copy_stream` and
 * return at once.  One fetch may be in flight per descriptor at a time; a
 * second fetch must be ordered after the first (same stream or an event).
 * opts = NULL selects the defaults (persistent, AUTO engine, auto grid, unpaced). */
OC_API int oc_fetch_layerwise(oc_desc* desc, const oc_fetch_opts* opts, void* copy_stream);

/* fetch_layers (Alg. A1's per-layer loop, split at the caller's layer
 * boundaries; the serving node's call order match -> descriptor -> layer waits,
 * P:720-729): the transfer of layers [l0, l1) only, so the consumer decides
 * when each part of the fetch runs (e.g. layer l+2 enqueued on a copy stream
 * that waits for the consumer's attention of layer l, so the copy co-runs with
 * that layer's MLP GEMMs instead of the attention).  l0 = 0 opens a new fetch
 * exactly like fetch_layerwise (same contract; it fixes the unit size) and
 * launches its first l1 layers; every later call continues it and must start
 * where the previous call stopped (l0 = previous l1).  Ranges may be enqueued on
 * different streams and may run concurrently; layers are still announced
 * (wait_layer, layers_ready, layer_times) strictly in order -- a range's layers
 * only after every earlier layer.  A new fetch of the descriptor must be
 * ordered after all ranges of the open one (as for fetch_layerwise).  A new fetch of the descriptor (any entry point) is refused
 * with EINVAL until all L layers of the open one have been requested.
 * opts: PERSISTENT mode, BULK or LDST engine (AUTO picks between them), unpaced;
 * max_ctas and OC_FETCH_LEAN apply per call; OC_FETCH_YIELD on a call with l0 > 0
 * and the BULK engine launches one copy CTA per unit (as the yield launch's later
 * layers); unit_bytes only with l0 = 0 (a later call may repeat the same value or
 * pass 0).  Errors: ERANGE (l0 >= l1 or l1 > L),
 * EINVAL (out of order), ENOTSUP (other modes, engines, pacing). */
OC_API int oc_fetch_layers(oc_desc* desc, uint32_t l0, uint32_t l1, const oc_fetch_opts* opts,
                           void* copy_stream);

/* scatter_flat -- the client half of the paper's unfused flow (Alg. A1 line 6 RDMA-writes B_l into
 * the client buffer; the client then copies it into its paged KV cache): a
 * layer-major payload at flat_base (device address, [L][N][S]: layer l, chunk j at
 * (l*N + j)*S, 16-byte aligned, flat_capacity >= N*L*S) is scattered into the descriptor's
 * target with the same per-layer completion as a fetch (wait_layer, layer_times).  opts: unit
 * size and copy-CTA cap (PERSISTENT, unpaced; ENOTSUP otherwise).  ERANGE / EALIGN as stated. */
OC_API int oc_scatter_flat(oc_desc* desc, uint64_t flat_base, uint64_t flat_capacity, const oc_fetch_opts* opts,
                           void* stream);

/* Batches: concurrent requests (P:467-598 treats them as tenants sharing one link) fetched by
 * ONE persistent launch.  Units are claimed in a single global order -- layer l of every request,
 * then layer l+1 -- so every request's layers arrive in order and all requests' early layers go
 * first.  Descriptors must share layout and device, and stay alive (not freed) until the batch
 * is freed.  Each member keeps its own layer-ready state: wait_layer / sync_layer / layer_times
 * work per descriptor as after fetch_layerwise.  PERSISTENT mode, unpaced only (ENOTSUP
 * otherwise); engine BULK, LDST or AUTO (LDST as soon as one member's target is head-split);
 * a batch may be fetched repeatedly, one fetch in flight at a time. */
typedef struct oc_batch oc_batch;
OC_API int oc_batch_create(oc_desc* const* descs, uint32_t n, oc_batch** out);
OC_API int oc_fetch_batch(oc_batch* batch, const oc_fetch_opts* opts, void* copy_stream);
OC_API int oc_batch_free(oc_batch* batch);

/* Order of a batch's units inside each layer (oc_fetch_batch; every order is layer-major, so every
 * request's layers arrive in order):
 *   BY_REQUEST  (default) request 0's units of layer l, then request 1's, ...;
 *   BY_POSITION blocks of B consecutive chunk positions (B*S ~ 4 MiB; env OC_BYPOS_BLOCK_KIB):
 *               block b of every member holding it (members in order of decreasing N, each
 *               member's B positions tile by tile), then block b+1.  Members that share a prefix
 *               -- the same chunk at the same position -- re-read each shared slice ~B*S bytes
 *               after the first read, while L2 still holds it, so HBM serves it once; a member's
 *               layer l completes only when the longest member's layer l does. */
enum { OC_BATCH_BY_REQUEST = 0, OC_BATCH_BY_POSITION = 1 };
OC_API int oc_batch_set_order(oc_batch* batch, int order);

/* Weighted deficit round robin dispatch (Alg. A2 lines 6-7: "Hold per-request
 * rates stable for this epoch. Dispatch layer payloads with weighted deficit round robin.").
 * The batch's requests become one claim order: each request's copy units in layer-major order
 * (its layers still complete in order), interleaved by deficit round robin with quantum
 * q_i = floor(Q * w_i / min_j w_j) bytes per round (reading c21), cut into claim entries of at
 * most E units that copy CTAs take in sequence.  With hold_rates, w_i are rates in bytes/s and
 * request i's entries are released no earlier than t0 + (its bytes in earlier entries) / w_i
 * (whole microseconds; never before the previous entry; reading c22), t0 = the launch's start. */
typedef struct {
    const double* weights;   /* [n] one per batch member, finite and > 0 (e.g. the epoch rates r_i) */
    uint64_t quantum_bytes;  /* Q: bytes per round of the lightest request; 0 = max(256 KiB,
                                largest unit); EINVAL if below the largest unit               */
    uint32_t entry_units;    /* E: units per claim entry; 0 = 8                               */
    uint32_t hold_rates;     /* 1: pace request i at weights[i] bytes/s                       */
    const uint64_t* free_units; /* [n] or NULL: leading units of request i read from an HBM
                                mirror (they never cross the paced link): they are claimed
                                first, request by request, released at t0, and DRR and the
                                held rates cover only the rest (reading c25);
                                oc_fetch_batch_wdrr fills it from the members' hot layers
                                when NULL                                                     */
    uint32_t layer_packets;  /* 0: a DRR packet is one copy unit (reading c21).  L (the model's
                                layer count): a packet is a request's whole layer payload,
                                N_i*S bytes -- Alg. A2 line 7 as written; n_units[i] must be
                                a multiple of L, free_units whole layers, Q >= the largest
                                payload (default max(256 KiB, largest payload)); EINVAL
                                otherwise                                                     */
} oc_wdrr_opts;

/* Fetch a batch in WDRR order (instead of layer-major across requests).  Same contract as
 * oc_fetch_batch; opts as there (PERSISTENT, BULK; pace_Bps must be 0 -- use hold_rates).
 * Errors: EINVAL (weights, quantum), ERANGE (a release time beyond 2^32 us, too many units). */
OC_API int oc_fetch_batch_wdrr(oc_batch* batch, const oc_fetch_opts* opts, const oc_wdrr_opts* wdrr,
                               void* copy_stream);

/* The claim order itself (host only; what oc_fetch_batch_wdrr uploads): n requests of
 * n_units[i] units, unit u of every request carrying tile_bytes[u % tiles] bytes.  Writes up to
 * `cap` entries (request, first unit, unit count, release us; any output pointer may be NULL)
 * and sets *n_entries (ERANGE if it exceeds cap). */
OC_API int oc_wdrr_plan(const uint64_t* n_units, uint32_t n, const uint32_t* tile_bytes, uint32_t tiles,
                        const oc_wdrr_opts* wdrr, uint32_t* ent_req, uint32_t* ent_first, uint32_t* ent_count,
                        uint32_t* ent_release_us, uint64_t cap, uint64_t* n_entries);

/* wait_layer (NotifyLayerReady, Alg. A1 line 7): make `consumer_stream` wait,
 * without blocking the host, until layer `layer` of the most recent fetch is
 * in place.  Layers become ready in increasing order.  For CHUNK_MAJOR
 * delivery every layer waits for the whole prefix (Eq. 2 chunkwise).
 * PERSISTENT mode: if the layer is already announced when the call is made (the
 * announcing kernel also writes a pinned host copy of the ready word, after the
 * device word), nothing is enqueued -- the bytes are already in place.
 * Otherwise a one-thread kernel that spins on the ready word goes on
 * `consumer_stream` (it holds one CTA slot, never a hardware queue).  Opt-in:
 * OC_WAIT_VALUE=1, a stream value wait (cuStreamWaitValue32) on `consumer_stream`;
 * OC_WAIT_RELAY=1, the value wait on a private relay stream + a CUDA event.  A
 * blocked value wait stalls the hardware queue its stream is mapped to, and streams
 * share queues (CUDA_DEVICE_MAX_CONNECTIONS): a producer mapped behind it waits too.
 * PER_LAYER mode: cudaStreamWaitEvent on the layer's event. */
OC_API int oc_wait_layer(oc_desc* desc, uint32_t layer, void* consumer_stream);

/* Host-blocking variant of wait_layer. */
OC_API int oc_sync_layer(oc_desc* desc, uint32_t layer);

/* layers_ready (NotifyLayerReady, Alg. A1 line 7, seen from the host):
 * *n = how many layers of the most recent fetch are announced, as
 * the host sees it now (non-blocking poll of the pinned copy of the ready word;
 * a layer counted here is in place in device memory).  PERSISTENT-mode fetches
 * (kernel and CE engines); for a PER_LAYER fetch, the layers whose CUDA event
 * has completed.  CHUNK_MAJOR delivery reports 0 or L.  EINVAL if no fetch was
 * issued; ENOTSUP if the descriptor has no host mirror (pinned allocation failed). */
OC_API int oc_layers_ready(oc_desc* desc, uint32_t* n);

/* Per-layer ready times of the most recent fetch, in ns of the GPU global
 * timer: out[0] = kernel start, out[1 + l] = layer l ready.  Blocks until the
 * fetch is complete.  `out` holds L + 1 values. */
OC_API int oc_layer_times(oc_desc* desc, uint64_t* out);

/* Asynchronous variant for pipelined callers: enqueues on `stream` a wait for
 * the most recent fetch's completion and a copy of its L + 1 stamps into `out`
 * (page-locked host or device memory, caller-owned; valid until `stream` has
 * passed the copy).  Returns at once; the caller synchronises on `stream` (or an
 * event recorded after this call) before reading `out`. */
OC_API int oc_layer_times_async(oc_desc* desc, uint64_t* out, void* stream);

/* Measurement support (not a step of the method): the compute window C_l of
 * the stall accounting (Eq. 3; a8).  Enqueues on `stream` (the
 * current device's) one single-CTA kernel that spins on the GPU global timer
 * for `ns` nanoseconds, leaving the other SMs to the fetch.  If `stamps` (a
 * device address, 8-byte aligned) is not NULL the kernel writes its start and
 * end time there (2 values, same clock as oc_layer_times).  ns > 60 s ->
 * OC_ERANGE. */
OC_API int oc_emulate_compute(uint64_t ns, uint64_t* stamps, void* stream);

/* Measurement support (not a step of the method): with the environment variable
 * OC_TRACE=1, every single-descriptor BULK launch records, per copy CTA b
 * (1 <= b < 2048), 8 GPU-global-timer stamps of its ramp: [0] CTA start,
 * [1] barriers initialised, [2] first claim returned, [3] first load issued,
 * [4] first unit in shared memory, [5] first unit's stores issued, [6] first
 * retire handed to the signaler, [7] signaler's first release published.
 * Copies the last traced launch's min(n, 2048*8) stamps (slot b*8+i; 0 =
 * not reached) into `out` (host).  Blocks until the device is idle. */
OC_API int oc_trace_read(uint64_t* out, uint64_t n);

/* ---- bandwidth scheduling (Sec. 3.6) --------------------------- */
typedef enum {
    OC_POL_EQUAL = 0,         /* B / n                                    */
    OC_POL_KV_PROP = 1,       /* proportional to s_i                      */
    OC_POL_BW_PROP = 2,       /* proportional to r_i* = s_i / c_i         */
    OC_POL_STALL_OPT = 3,     /* Eq. 6, caps r_i*                         */
    OC_POL_CAL_STALL_OPT = 4, /* Eq. 7 + Alg. A2, caps r_i* + delta       */
} oc_policy;

typedef struct {
    double bytes_per_layer;      /* s_i (bytes)   */
    double compute_per_layer_s;  /* c_i (seconds) */
} oc_profile;

/* schedule_bandwidth: per-request rates (bytes/s) under the shared cap B.
 * Stall-opt solves min sum s_i/r_i s.t. sum r_i = B, 0 < r_i <= cap_i by
 * capped water-filling (r_i = min(cap_i, lambda*sqrt(s_i)), reading c8); if
 * the caps fit in B each request gets its cap and the rest stays unused
 * (reading c10).  EINVAL if B <= 0, delta < 0, or some s_i/c_i <= 0; n = 0 is
 * OK.  Pure and thread-safe. */
OC_API int oc_schedule_bandwidth(int policy, const oc_profile* profiles, uint64_t n, double cap_Bps,
                                 double delta_Bps, double* rates_out);

/* ---- multi-tenant pool: epoch admission (Sec. 3.4; Sec. 3.6; Alg. A2) -----
 * submit: a request (its descriptor, per-layer compute window c_i and copy stream) joins the
 *   pool.  If W = N*L*S < theta (Eq. 2) it is served chunkwise at once, unpaced and outside the
 *   pool (state CHUNKWISE); otherwise it waits for the next epoch (state WAITING).
 * epoch: requests whose fetch has finished leave (their bandwidth returns now, not earlier);
 *   every waiting request is admitted with a rate from schedule_bandwidth(policy, s_i = N*S,
 *   c_i, cap - rates still in use, delta) and its fetch is launched paced at that rate for the
 *   whole load (state RUNNING).  No admission when nothing is left of the cap.
 * set_dispatch: INDEPENDENT (default) launches each admitted request as its own fetch paced at
 *   its rate; WDRR launches the epoch's admitted requests as one oc_fetch_batch_wdrr with weights
 *   = rates and hold_rates = 1 (Alg. A2 lines 6-7) on the first admitted request's stream.
 * The descriptors must outlive the pool's use of them.  Not thread-safe across pools sharing a
 * descriptor. */
typedef struct oc_tenant_pool oc_tenant_pool;
enum { OC_TENANT_WAITING = 0, OC_TENANT_RUNNING = 1, OC_TENANT_DONE = 2, OC_TENANT_CHUNKWISE = 3 };
OC_API int oc_pool_create(int policy, double cap_Bps, double delta_Bps, uint64_t theta_bytes, oc_tenant_pool** out);
enum { OC_DISPATCH_INDEPENDENT = 0, OC_DISPATCH_WDRR = 1 };
OC_API int oc_pool_set_dispatch(oc_tenant_pool* pool, int dispatch);
OC_API int oc_pool_submit(oc_tenant_pool* pool, oc_desc* desc, double compute_per_layer_s, void* copy_stream,
                          uint64_t* ticket);
OC_API int oc_pool_epoch(oc_tenant_pool* pool, uint64_t* n_admitted);
OC_API int oc_pool_status(oc_tenant_pool* pool, uint64_t ticket, int* state, double* rate_Bps);
OC_API int oc_pool_destroy(oc_tenant_pool* pool);

/* ---- errors ---------------------------------------------------------------- */
OC_API const char* oc_last_error(void);
OC_API const char* oc_status_str(int status);
OC_API int oc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* OBJCACHE_H */
