/* trims.h — C ABI of the B200-native TrIMS model store (libtrims.so).
 *
 * This is the drop-in boundary for the reference's load-and-serve path
 * (SURVEY.md §8b). Plain pointers, sizes and ints only; every function
 * returns 0 or a reference Errc value (proj/include/mrm/error.hpp:11-56;
 * wire codes 1..7 unchanged) and never lets a C++ exception cross the ABI.
 * trims_last_error() returns the thread's last failure message.
 *
 * Each entry point names the reference interface it replaces (file:line,
 * relative to /root/reference). INTEGRATION.md shows how a maintainer binds
 * it from the reference side (C++ TierBackend subclass / client SDK shim).
 */
#ifndef TRIMS_H
#define TRIMS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */

/* error.cpp:5-38 errc_name */
const char* trims_errc_name(int code);
/* error.cpp:41-69 wire_code: collapse a fine code onto wire codes 1..7 */
int trims_wire_code(int code);
/* thread-local detail of the last non-zero return */
const char* trims_last_error(void);
/* library / device facts: cuda device count (0 on GPU-less hosts), SHA-NI use */
int trims_device_count(void);
/* Create the device's primary context ahead of the first open/attach. */
int trims_device_init(int device);
int trims_sha_hw(void);

/* ------------------------------------------------- artifact format (a1, a2, a7) */

/* Sha256::of (proj/src/sha256.cpp:24-123) */
int trims_sha256(const void* data, uint64_t n, uint8_t out[32]);

/* model::read_manifest(path, full_verify) (model_format.cpp:370-409).
 * json_out gets the canonical manifest JSON (nlohmann dump() bytes). */
int trims_read_manifest(const char* path, int full_verify, char* json_out, uint64_t cap,
                        uint8_t checksum_out[32], uint64_t* blob_bytes, uint64_t* blob_file_offset);

/* model::manifest_from_json -> manifest_to_json round trip (model_format.cpp:179-229) */
int trims_manifest_canonical(const char* json_in, char* json_out, uint64_t cap);

/* model::make_manifest (model_format.cpp:158-177). decls: "name dtype d0,d1,...\n" */
int trims_make_manifest(const char* ns, const char* name, const char* version, const char* decls,
                        uint64_t workspace_bytes, char* json_out, uint64_t cap);

/* model::write_model_file (model_format.cpp:293-305): blob = full blob_bytes
 * (padding included) of the manifest. */
int trims_write_model(const char* path, const char* manifest_json, const void* blob);

/* shm::layout_for (shared_segment.cpp:63-95). kind 0 model, 1 layer, 2 block.
 * Output lines "name segment offset length\n". */
int trims_layout_for(const char* manifest_json, uint32_t kind, uint64_t block_bytes, char* out,
                     uint64_t cap);

/* The ingest plan (new: the reference keeps artifact bytes verbatim).
 * flags bit0 = convert floating tensors to out_dtype, bit1 = KCRS->KRSC for
 * 4-D tensors. out_dtype uses the manifest dtype codes: 0 f64 1 f32 2 f16
 * 3 i8 4 bf16. Writes the resident manifest JSON. */
#define TRIMS_PLAN_CONVERT 1u
#define TRIMS_PLAN_PERMUTE_4D 2u
int trims_resident_manifest(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, char* json_out,
                            uint64_t cap);

/* ---------------------------------- synthetic weights (a12, K5), host side */

/* bench::gen_catalog inner loop (catalog.cpp:143-154): n splitmix64 words of
 * stream `stream_seed` starting at element k0 (multi-threaded). */
int trims_fill_splitmix_host(uint64_t* dst, uint64_t n, uint64_t stream_seed, uint64_t k0);
/* uniform fp32 init fmaf(hi-lo, u24*2^-24, lo) (our definition, K5) */
int trims_fill_uniform_host(float* dst, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi);
/* bench::fnv1a (catalog.cpp:79-86) */
uint64_t trims_fnv1a(const char* s);
/* Client::touch (client.cpp:338-359) over a host blob + manifest */
int trims_touch_host(const void* blob, const char* manifest_json, uint64_t* out);
/* TRIMS block checksum over a host buffer (CPU twin of the device K4) */
int trims_checksum_host(const void* p, uint64_t n, uint64_t word0, uint64_t* out);

/* --------------------------------------------- the store (CacheCore + CudaTierBackend) */

typedef struct trims_store trims_store;

typedef struct trims_store_config {
  uint64_t fast_capacity_bytes;  /* daemon.hpp:21 (HBM budget, logical bytes) */
  uint64_t host_capacity_bytes;  /* daemon.hpp:22 (pinned DRAM budget) */
  uint64_t disk_capacity_bytes;  /* daemon.hpp:24 */
  uint32_t policy;               /* 0 LRU, 1 LCU (daemon.hpp:26) */
  uint32_t eager_reclaim;        /* daemon.hpp:27 */
  uint32_t full_verify;          /* daemon.hpp:32 */
  int32_t device;                /* CUDA ordinal of this store's fast tier */
  const char* disk_cache_dir;    /* daemon.hpp:23 */
  uint32_t plan_flags;           /* TRIMS_PLAN_* (0 = bytes verbatim, reference behaviour) */
  uint32_t out_dtype;            /* target dtype when TRIMS_PLAN_CONVERT */
  uint64_t pinned_pool_bytes;    /* pre-pinned host pool (0 = host_capacity_bytes) */
  uint32_t scan_disk;            /* register *.trms in disk_cache_dir at start (daemon.cpp:314-325) */
  uint32_t read_threads;         /* parallel pread threads for disk -> pinned (0 = 8) */
  uint64_t arena_bytes;          /* HBM arena of the fast tier: 0 = auto, 1 = off (one cuMem allocation per model) */
  /* Multi-GPU (no reference counterpart — the reference runs
   * one daemon per node): one store per GPU process, all sharing a node-local
   * residency directory. A fast-tier miss whose model is sealed on a peer GPU
   * is served by an NVLink pull of the peer's segment (TRIMS_PEER_HIT). */
  const char* directory;         /* /dev/shm name shared by the node's stores; NULL = single GPU */
  int32_t rank;                  /* this store's row in the directory */
  int32_t world;                 /* stores on the node */
  uint32_t directory_slots;      /* per-rank slots (0 = 1024) */
  const char* remote_url;        /* daemon.hpp:26: http://... or dir:<path>; NULL = no remote tier */
  double workspace_headroom_fraction; /* daemon.hpp:29 (in [0, 1]; published in stats for the client's
                                         workspace-reservation fallback, client.cpp:192-204) */
  uint32_t startup_calibration;  /* daemon.hpp:33: measure q/o/s at creation (daemon.cpp:342-390) */
  /* Cold loads read the artifact with O_DIRECT straight into the pinned host
   * tier (no page-cache copy): 0 = buffered reads, 1 = direct, 2 = auto
   * (direct when most of the blob is not in the page cache). Filesystems
   * without O_DIRECT fall back to buffered reads. */
  uint32_t direct_io;
  /* Multi-GPU: a fast-tier miss held by a peer rank is served IN PLACE (the
   * peer's segment mapped read-only here, its range leased from the holder)
   * instead of copied (1), outcome TRIMS_PEER_MAP; 0 = copy (PeerHit). In-process
   * opens (trims_store_open); the daemon's opens keep PeerHit copies. */
  uint32_t peer_map;
} trims_store_config;

/* Reference outcomes (cache_core.hpp:36) + PEER_HIT for the multi-GPU directory. */
enum { TRIMS_FAST_HIT = 0, TRIMS_HOST_HIT = 1, TRIMS_DISK_LOAD = 2, TRIMS_REMOTE_FETCH = 3, TRIMS_PEER_HIT = 4,
       TRIMS_PEER_MAP = 5 };

/* One open's result: PlacementResult (cache_core.hpp:48-57) + the exported
 * segment (ExportedSegment cache_core.hpp:59-63 / wire ObjectRef
 * wire_protocol.hpp:44-62) carrying a cuMem POSIX-fd instead of a shm name. */
typedef struct trims_export {
  uint64_t model_id;
  uint32_t outcome;
  int32_t device;
  uint64_t generation;
  uint64_t payload_bytes;         /* resident blob + JSON + 8 */
  uint64_t resident_blob_bytes;
  uint64_t alloc_bytes;           /* physical cuMem allocation (granularity-rounded) */
  uint64_t weights_bytes;         /* artifact footprint (accounting unit) */
  uint64_t workspace_bytes;
  uint64_t ingest_checksum;       /* TRIMS block checksum of the resident blob */
  uint64_t timings_ns[4];         /* fetch, disk_read, host_to_fast_copy, handle_export */
  uint8_t manifest_digest[32];    /* SHA-256 of the resident manifest JSON */
  void* dev_ptr;                  /* owner-process device address */
  int32_t fd;                     /* owner-process fd of the allocation (the arena, or a dedicated segment) */
  uint32_t n_objects;             /* layout_for(resident manifest, granularity) count */
  char token[160];                /* names the allocation: one token per arena */
  uint64_t segment_offset;        /* segment start inside that allocation */
} trims_export;

/* ---- The TierBackend seam itself (cache_core.hpp:76-98): the eight virtuals
 * of the reference's plugin, implemented by CudaTierBackend, for a reference
 * CacheCore/daemon to drive directly (INTEGRATION.md shows the adapter).
 * Manifests cross as their canonical JSON; the trailer checksum separately. */
typedef struct trims_backend trims_backend;
int trims_backend_create(const trims_store_config* cfg, trims_backend** out);
void trims_backend_destroy(trims_backend* b);
/* ShmTierBackend::locate (daemon.cpp:128-136): DiskCache = the path; Remote
 * (not on disk, remote_url set) = rc 0 with an empty path; NotFound when absent. */
int trims_backend_locate(trims_backend* b, const char* ns, const char* name, const char* version, char* path_out,
                         uint64_t cap, uint64_t* file_bytes);
/* ShmTierBackend::fetch_remote (daemon.cpp:138-142): remote tier -> disk cache */
int trims_backend_fetch_remote(trims_backend* b, const char* ns, const char* name, const char* version,
                               char* path_out, uint64_t cap, uint64_t* file_bytes);
/* ShmTierBackend::read_manifest (daemon.cpp:144-151). With full_verify the
 * verified blob stays in pinned memory for the same key's stage_host /
 * publish_fast (read once, hashed once); trims_backend_load_settled drops it
 * if the open fails in between (our CacheCore calls it when a load settles). */
int trims_backend_read_manifest(trims_backend* b, const char* ns, const char* name, const char* version,
                                const char* path, char* json_out, uint64_t cap, uint8_t checksum_out[32]);
/* ShmTierBackend::stage_host (daemon.cpp:153-158): disk -> pinned host tier */
int trims_backend_stage_host(trims_backend* b, uint64_t model_id, const char* manifest_json,
                             const uint8_t checksum[32], const char* path);
/* ShmTierBackend::publish_fast (daemon.cpp:160-209): -> HBM arena segment, exported */
int trims_backend_publish_fast(trims_backend* b, uint64_t model_id, const char* manifest_json, int from_host,
                               const char* path, trims_export* out);
/* ShmTierBackend::evict_fast/host/disk (daemon.cpp:211-224) */
int trims_backend_evict_fast(trims_backend* b, uint64_t model_id);
int trims_backend_evict_host(trims_backend* b, uint64_t model_id);
int trims_backend_evict_disk(trims_backend* b, const char* path);
int trims_backend_load_settled(trims_backend* b, const char* ns, const char* name, const char* version);

/* remote::fetch(make_ref(url, key), dest_dir) (remote_store.cpp:58-120): a
 * dir:<path> / bare-path store is copied, http://host[:port][/prefix] is
 * fetched by HTTP/1.1 GET; the download must pass a full verify before it is
 * renamed to <dest_dir>/<ns>__<name>__<version>.trms. RemoteNotFound,
 * TransportError, ChecksumMismatch. Host only (no device). */
int trims_remote_fetch(const char* url, const char* ns, const char* name, const char* version, const char* dest_dir,
                       char* path_out, uint64_t cap, uint64_t* file_bytes);

/* Daemon::Daemon (daemon.cpp:298-391) minus listeners: builds the backend
 * and the core, optionally scans the disk cache. */
int trims_store_create(const trims_store_config* cfg, trims_store** out);
void trims_store_destroy(trims_store* s); /* Daemon::join: drop_all (daemon.cpp:597) */

/* Daemon::handle_open -> CacheCore::open_model (daemon.cpp:452-476,
 * cache_core.cpp:194-423). The logical clock advances per open. */
int trims_store_open(trims_store* s, const char* ns, const char* name, const char* version,
                     uint32_t gran_kind, uint64_t block_bytes, trims_export* out);
/* CacheCore::close_model (cache_core.cpp:425-445) */
int trims_store_close(trims_store* s, const char* ns, const char* name, const char* version,
                      uint64_t* refcount_out);
/* CacheCore::reclaim (cache_core.cpp:168-171); evicted keys as "ns/name@ver\n" */
int trims_store_reclaim(trims_store* s, uint32_t tier, uint64_t bytes, uint32_t policy, char* out,
                        uint64_t cap);
/* CacheCore::register_disk_file (cache_core.cpp:474-485) */
int trims_store_register_disk_file(trims_store* s, const char* ns, const char* name,
                                   const char* version, const char* path, uint64_t bytes);
/* CacheCore::drop_all (cache_core.cpp:512-529) */
int trims_store_drop_all(trims_store* s);
/* CacheCore::stats (cache_core.cpp:447-472) as a JSON document. */
int trims_store_stats_json(trims_store* s, char* out, uint64_t cap);
/* The resident manifest JSON of a fast-resident model. */
int trims_store_resident_json(trims_store* s, uint64_t model_id, char* out, uint64_t cap);
/* Last ingest of a model: h2d_ms, total_ms, read_ms, h2d_bytes, launches,
 * segment alloc_ms (cuMem create/map/export), seal_ms (tail + digest). */
int trims_store_ingest_stats(trims_store* s, uint64_t model_id, double out7[7]);
/* Per-tensor block checksums of a resident model (buckets = tensors + 1). */
int trims_store_checksums(trims_store* s, uint64_t model_id, uint64_t* out, uint64_t cap, uint64_t* n);
/* Is the model fast-resident in this store (no state change)? */
int trims_store_fast_resident(trims_store* s, const char* ns, const char* name, const char* version, int* out);

/* ------------------------------------------- multi-GPU residency directory */

/* One sealed fast-tier segment as published for peers. */
typedef struct trims_dir_coords {
  int32_t rank, device, pid, fd;  /* owner rank / GPU / process, and its fd of the exportable allocation */
  uint32_t arena, reserved;       /* arena: the allocation outlives the segment */
  uint64_t alloc_bytes, offset;   /* allocation size; segment offset inside it */
  uint64_t payload_bytes, resident_blob_bytes, generation, checksum;
} trims_dir_coords;

typedef struct trims_dir trims_dir;
/* Create or attach the node directory `name` for world x slots; clears `rank`'s row. */
int trims_dir_open(const char* name, int world, int rank, uint32_t slots, trims_dir** out);
void trims_dir_close(trims_dir* d); /* clears this rank's row */
int trims_dir_unlink(const char* name);
int trims_dir_publish(trims_dir* d, const char* ns, const char* name, const char* version, const trims_dir_coords* c);
int trims_dir_retract(trims_dir* d, const char* ns, const char* name, const char* version);
/* Other ranks' live copies, best peer first (rendezvous order). */
int trims_dir_holders(trims_dir* d, const char* ns, const char* name, const char* version, trims_dir_coords* out,
                      uint64_t cap, uint64_t* n);
/* Rendezvous weight of (key "ns/name@version", rank). */
uint64_t trims_peer_score(const char* key, int rank);

/* --------------------------------------------------- client attach (a5, a9) */

typedef struct trims_import trims_import;
/* Maps an allocation exported by another (or this) process read-only — the
 * device side of Attachment::attach (shared_segment.cpp:212-245). fd must be
 * valid in the caller (SCM_RIGHTS / same process). With the arena, a client
 * maps once and attaches every model by offset. */
int trims_import_open(int device, int fd, uint64_t alloc_bytes, trims_import** out, void** base);
/* Attaches one model segment of a mapping: validates the tail (magic,
 * generation -> StaleGeneration, sealed, length), re-checks the manifest
 * digest (client.cpp:284-291), returns the device pointer and the resident
 * manifest JSON (client.cpp:293-307). */
int trims_import_attach(trims_import* im, uint64_t offset, uint64_t generation, uint64_t payload_bytes,
                        const uint8_t digest[32], void** dev_ptr, char* json_out, uint64_t cap);
int trims_import_read_only(trims_import* im);
/* Device-side integrity check of an attached segment: K4 over the resident
 * blob, compared with the checksum sealed into the tail (Corrupt if not). */
int trims_import_verify(trims_import* im, uint64_t offset, uint64_t generation, uint64_t payload_bytes,
                        uint64_t* checksum_out);
void trims_import_close(trims_import* im);

/* View lifetime (shared_segment.cpp:212-245 + test_shared_segment.cpp:99-110:
 * an attached view survives the owner's destruction of the segment). With
 * every model in one HBM arena, a reader holds the range it reads:
 *  - in the store's process, a pin keeps the published record (and its arena
 *    range) alive after eviction until released;
 *  - in another process, a lease row in the arena's shared lease table
 *    ("/<token>.leases") keeps the owner from reusing the range until it is
 *    released or the reader dies. Acquire while the model is open (the open
 *    handle guarantees the generation is current). A token without a lease
 *    table (a dedicated segment) yields *out = NULL: the mapping itself keeps
 *    the pages alive. */
typedef struct trims_pin trims_pin;
typedef struct trims_lease trims_lease;
int trims_store_pin(trims_store* s, uint64_t model_id, uint64_t generation, trims_pin** out);
void trims_pin_release(trims_pin* p);
int trims_lease_acquire(const char* token, uint64_t offset, uint64_t generation, trims_lease** out);
void trims_lease_release(trims_lease* l);

/* ------------------------------------------- ingest kernels (K1..K5) raw */

/* Pinned/pageable host raw blob -> resident blob on the device (what
 * publish_fast runs; daemon.cpp:160-209 + new convert/permute/checksum). */
int trims_ingest_host(int device, const void* host_blob, const char* src_json, uint32_t plan_flags,
                      uint32_t out_dtype, void* dev_dst, uint64_t* checksum_out, double stats_out5[5]);
/* HBM-resident raw blob -> resident blob, async on `stream` (cudaStream_t).
 * Bucket sums are accumulated into d_sums (must be zeroed by the caller). */
int trims_transform_device(int device, const void* dev_src, const char* src_json, uint32_t plan_flags,
                           uint32_t out_dtype, void* dev_dst, unsigned long long* d_sums, void* stream);
/* Compiled ingest plans: the tile table is built and uploaded once, so the
 * per-call host cost of the two entry points below is a few microseconds. */
typedef struct trims_plan trims_plan;
int trims_plan_create(int device, const char* src_json, uint32_t plan_flags, uint32_t out_dtype, trims_plan** out);
void trims_plan_destroy(trims_plan* p);
/* tiles, buckets, algo read bytes, algo write bytes, src blob, resident blob, chunks,
 * kernel launches per HBM-resident transform */
int trims_plan_describe(trims_plan* p, uint64_t out8[8]);
int trims_plan_resident_json(trims_plan* p, char* out, uint64_t cap);
int trims_plan_transform(trims_plan* p, const void* dev_src, void* dev_dst, unsigned long long* d_sums, void* stream,
                         uint32_t* launches);
int trims_plan_ingest_host(trims_plan* p, const void* host_blob, void* dev_dst, uint64_t* checksum_out,
                           double stats_out5[5]);
/* Roofline accounting of a plan: tiles, buckets, algorithmic read/write bytes. */
int trims_plan_info(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, uint64_t out4[4]);
/* TRIMS block checksum of a device range (async, accumulates into *d_out). */
int trims_checksum_device(const void* dev, uint64_t nbytes, uint64_t word0, unsigned long long* d_out,
                          void* stream);
/* The GPU compute step of a catalog request (the role of Client::touch,
 * client.cpp:338-359): the block checksum of `nbytes` at `dev` on a stream of
 * the calling thread, synchronously; *out = the sum (every byte read once). */
int trims_touch_device(int device, const void* dev, uint64_t nbytes, uint64_t* out);
/* K5 on device: splitmix words / uniform fp32 (bit-identical to the host fills). */
int trims_fill_splitmix_device(uint64_t* dev, uint64_t n, uint64_t stream_seed, uint64_t k0, void* stream);
int trims_fill_uniform_device(float* dev, uint64_t n, uint64_t stream_seed, uint64_t j0, float lo, float hi,
                              void* stream);

/* ------------------------------------------- forward pass (K7, K8) */

/* K7: D[M,N] = relu?(A[M,K] . B[N,K]^T * scale[n] + bias[n] + residual[m,n]),
 * bf16 operands (row strides lda/ldb/ldd/ldr in elements, 16-byte aligned),
 * fp32 accumulation in TMEM via tcgen05.mma; scale/bias/residual nullable.
 * bn = output tile width 64/128/256 or 0 (auto). Async on `stream`. */
int trims_gemm_bf16(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N, uint64_t ldb,
                    void* D, uint64_t ldd, const float* scale, const float* bias, const void* residual, uint64_t ldr,
                    int relu, int bn, void* stream);
/* The same with an explicit split-K count: splits = 1, 2, 4 or 8 (the S
 * splits of an output tile run as one thread-block cluster and reduce their
 * fp32 partials in split order through distributed shared memory), or 0 to
 * pick it as the network executor does. */
int trims_gemm_bf16_split(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N,
                          uint64_t ldb, void* D, uint64_t ldd, const float* scale, const float* bias,
                          const void* residual, uint64_t ldr, int relu, int bn, int splits, void* stream);
/* The same with weight multicast: mc = 1, 2, 4 or 8 consecutive M-tiles form
 * one thread-block cluster dimension and share every weight (B) stage by TMA
 * multicast (splits * mc <= 8; bn 64 or 128); mc = -2: a 2-SM pair, tcgen05
 * cta_group::2 MMAs of M = 256 over two CTAs that each load half of B
 * (splits 1; bn 128 or 256); mc = -3: persistent (one CTA per SM over all
 * output tiles, two TMEM accumulators so a tile's epilogue overlaps the next
 * tile's k-loop; splits ignored, 16-byte aligned output rows). */
int trims_gemm_bf16_ex(const void* A, uint64_t M, uint64_t K, uint64_t lda, const void* B, uint64_t N, uint64_t ldb,
                       void* D, uint64_t ldd, const float* scale, const float* bias, const void* residual,
                       uint64_t ldr, int relu, int bn, int splits, int mc, void* stream);

/* The compute on shared weights (replaces Client::touch, client.cpp:338-359):
 * a CNN bound to a resident manifest whose bf16 KRSC weights start at
 * `weights` (an attached segment). arch_text: one layer per line (written by
 * paper_1811_09732_b200/models.py). The net owns its workspace, an fp32 NCHW
 * input buffer and an fp32 logits buffer. */
typedef struct trims_net trims_net;
int trims_net_create(int device, const char* arch_text, const char* resident_json, const void* weights, int batch,
                     trims_net** out);
/* The same with executor flags: TRIMS_NET_THROUGHPUT (1) builds no split-K
 * launches (one CTA per output tile) so many clients' forwards pack the GPU;
 * TRIMS_NET_LEAN (2) also uses GEMM variants that fit two CTAs per SM.
 * 0 = latency mode (trims_net_create). */
#define TRIMS_NET_THROUGHPUT 1
#define TRIMS_NET_LEAN 2
int trims_net_create_ex(int device, const char* arch_text, const char* resident_json, const void* weights, int batch,
                        int flags, trims_net** out);
void trims_net_destroy(trims_net* net);
int trims_net_buffers(trims_net* net, void** input, void** logits, int* classes, int* input_hw);
/* Re-point a net at a new generation of the same resident model (after an
 * eviction + reload): only weight-dependent state is rebuilt. */
int trims_net_rebind(trims_net* net, const void* weights);
/* One forward pass, async on `stream`; use_graph replays a captured CUDA graph. */
int trims_net_run(trims_net* net, void* stream, int use_graph);
/* flops per forward, kernel launches per forward, workspace bytes */
int trims_net_info(trims_net* net, double out3[3]);
/* One request end to end on `stream`: host input (fp32 NCHW, batch x 3 x H x W)
 * -> device, forward, logits (fp32 batch x classes) -> host, synchronised.
 * Pinned host buffers give the full PCIe rate. */
int trims_net_forward_host(trims_net* net, const float* host_input, float* host_logits, void* stream, int use_graph);
/* Page-locked host memory for request buffers (a pageable input makes every
 * H2D a CPU-side staging copy: with many client processes the host cores,
 * not the GPU, become the bound). */
int trims_host_alloc(uint64_t bytes, void** out);
void trims_host_free(void* p);
/* Parity tap: the device buffer architecture layer `layer` (0-based, the
 * input line excluded) wrote in the last forward, NHWC dims4 = {n, h, w, c},
 * dtype 0 = bf16, 1 = fp32 (the logits), 2 = not kept (a conv whose 2x2 max
 * pool ran in its epilogue: *ptr = NULL, the pool layer's tap holds the
 * pooled result). layer < 0 returns the layer count.
 * No reference counterpart (the reference has no inference math); it lets the
 * tests check every layer against the CPU oracle on the device's own inputs. */
int trims_net_tap(trims_net* net, int layer, const void** ptr, int dims4[4], int* dtype);
/* row softmax of fp32 logits [M, N] (device pointers) */
int trims_softmax(const float* in, float* out, int M, int N, void* stream);

/* Host-only view of an ingest plan's tile schedule (no device needed): one
 * "tile op src_off dst_off dst_bytes n_elem tensor" line per logical tile of
 * the kernel-grouped table, then per group "group kind tiles nbins stride tail
 * dev_begin dev_count" followed by its device-image entries ("dev ..."; op 255
 * = bin padding). For tests of the static-bin + dynamic-tail scheduler. */
int trims_tile_plan_text(const char* src_json, uint32_t plan_flags, uint32_t out_dtype, int sm_count, char* out,
                         uint64_t cap);

/* ------------------------------------------------------------ daemon
 * The wire-protocol server (proj/src/daemon.cpp:398-560 over
 * proj/src/wire_protocol.cpp's frozen v1 frames): serves OpenRequest /
 * CloseRequest / StatsRequest for `store` on endpoint "unix:<path>" (or a bare
 * path) / "tcp:<ipv4>:<port>", one thread per connection; handles still open
 * when a connection drops are closed. OpenResponse objects tile the resident
 * blob; each ObjectRef token is "<allocation>?dev=&alloc=&seg=&payload=" and,
 * on Unix sockets, the allocation's fd rides the frame (SCM_RIGHTS).
 * Replaces mrm::daemon::Daemon::start/request_stop/join (daemon.hpp:77-131). */
typedef struct trims_server trims_server;
int trims_server_start(trims_store* store, const char* endpoint, trims_server** out);
void trims_server_stop(trims_server* s);
uint64_t trims_server_frames_served(trims_server* s);
/* v1 codec (wire_protocol.hpp:151-158 encode/decode) over a one-line text
 * form of a message, for parity tests against the reference's codec. */
int trims_wire_encode_text(const char* text, uint8_t* out, uint64_t cap, uint64_t* n);
int trims_wire_decode_text(const uint8_t* frame, uint64_t n, char* out, uint64_t cap);

/* ------------------------------------------------------------ test hooks */

/* Replays a decision trace through this library's CacheCore over an
 * in-memory backend (the reference FakeBackend contract, oracle.cpp:14-91).
 * Same spec / output text as oracle/ref_shim.cpp:ref_replay's "live" lines. */
int trims_replay(const char* spec, char* out, uint64_t cap);

/* One rank of a simulated node: the same CacheCore + open_with_peers as a
 * store, over the in-memory backend of trims_replay, publishing to a real
 * directory. spec = the "cfg" and "model" lines of a replay spec. step: kind
 * 'o' (open through the directory) or 'c' (close) of model i at clock `now`;
 * writes "<outcome> <fast_used> <host_used> <refcount> <peer_rank>". */
typedef struct trims_simcore trims_simcore;
int trims_simcore_create(const char* spec, const char* directory, int world, int rank, trims_simcore** out);
void trims_simcore_destroy(trims_simcore* c);
int trims_simcore_step(trims_simcore* c, char kind, uint32_t model, uint64_t now, char* out, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* TRIMS_H */
