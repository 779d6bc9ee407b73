/*
 * rise_b200.h — C ABI of the B200 (sm_100a) execution backend for RISE/Shine.
 *
 * This is the drop-in boundary that replaces the reference's execution stage
 * for emitted kernels.  In the reference (pure Python, package `risec`):
 *
 *   codegen.emit(unit, target)                -> kernel text      (codegen.py:451)
 *   cexec.execute_kernel(source, arguments)   -> runs the text    (cexec.py:509)
 *   cexec.run_emitted(code, unit, nats, ins)  -> nested result    (cexec.py:555)
 *
 * Here the kernel text is CUDA C++ for sm_100a, compiled at run time with
 * NVRTC, and executed through the entry points below.  The Python side
 * (`paper_2201_03611_b200.runtime`) binds them with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions (mirroring the reference's error model, errors.py:10-80):
 *   - every function returns int status: 0 = ok, nonzero = failure;
 *   - the failure text is available from rs_last_error() (thread-local);
 *   - the Python wrapper raises EmitError (stage "emit") for compile
 *     failures and InterpreterError (stage "run") for launch / memory
 *     failures, exactly the classes the reference raises from emit()
 *     (codegen.py:453-454) and execute_kernel() (cexec.py:516, 376, 495).
 *   - plain pointers and sizes only; no torch types cross this boundary.
 *   - device pointers are CUdeviceptr values carried as void*; streams and
 *     events are CUstream / CUevent handles carried as void*.  The runtime
 *     runs in the device's primary context, so buffers allocated by any
 *     other user of the primary context (e.g. PyTorch) are valid arguments.
 */
#ifndef RISE_B200_H
#define RISE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rs_module_s* rs_module;
typedef struct rs_function_s* rs_function;

/* ---- status / device ------------------------------------------------- */

/* Thread-local text of the last failure (never NULL). */
const char* rs_last_error(void);

/* ABI version of this library (bumped on any signature change). */
int rs_abi_version(void);

/* Load the CUDA driver (dlopen libcuda.so.1), init it and make `device`'s
 * primary context current on the calling thread.  Idempotent.
 * Replaces: nothing in the reference — cexec has no device (cexec.py:36-43
 * sequentialises the device id intrinsics instead). */
int rs_init(int device);

int rs_device_count(int* count);

/* CUdevice_attribute query on the current device (e.g. 16 = SM count). */
int rs_device_attribute(int attribute, int* value);

/* NVRTC version, for the build report. */
int rs_nvrtc_version(int* major, int* minor);

/* ---- compilation (replaces cexec.parse_kernel, cexec.py:97) ---------- */

/* Compile CUDA C++ `source` with NVRTC for sm_100a into a CUBIN and load it.
 * `opts` are NVRTC options (the architecture option is added if absent).
 * `name_exprs` are the kernel name expressions to instantiate (template
 * kernels such as "mvKernel<8192, 8192>"); their lowered (mangled) names are
 * available through rs_module_lowered_name in the same order.
 * Compile failure: status != 0 and the NVRTC log in rs_last_error(). */
int rs_compile(const char* source, const char* program_name,
               const char* const* opts, int nopts,
               const char* const* name_exprs, int nexprs,
               rs_module* out_module);

/* Compile only (no device needed): returns the CUBIN image in a buffer owned
 * by the caller-visible handle; used by build() and the CPU test-suite. */
int rs_compile_cubin(const char* source, const char* program_name,
                     const char* const* opts, int nopts,
                     const char* const* name_exprs, int nexprs,
                     void** out_image, size_t* out_size,
                     char** out_lowered_names /* '\n'-separated, malloc'd */,
                     char** out_log /* malloc'd */);
void rs_free_host(void* p);

/* Load a previously compiled CUBIN image (on-disk cache). */
int rs_module_load(const void* image, size_t size, rs_module* out_module);

int rs_module_lowered_name(rs_module m, int index, const char** out_name);
int rs_module_get_function(rs_module m, const char* lowered_name, rs_function* out_fn);
int rs_module_unload(rs_module m);

/* CUfunction_attribute query (e.g. 4 = NUM_REGS, 1 = SHARED_SIZE_BYTES). */
int rs_function_attribute(rs_function f, int attribute, int* value);

/* ---- launch (replaces cexec.execute_kernel's _exec_block, cexec.py:526) */

/* Launch `f` with grid/block dims, an optional thread-block-cluster shape
 * (cluster == NULL or {1,1,1} for none), `smem` bytes of dynamic shared
 * memory (the >48 KB opt-in attribute is set automatically) on `stream`
 * (NULL = legacy default stream).  `args` follows cuLaunchKernel's
 * kernelParams convention: an array of pointers to each argument value. */
int rs_launch(rs_function f, const unsigned grid[3], const unsigned block[3],
              const unsigned cluster[3], unsigned smem, void* stream, void** args);

/* rs_launch with launch flags: RS_LAUNCH_COOPERATIVE (all blocks co-resident,
 * for kernels with grid-wide barriers; the launch fails rather than hangs
 * when the grid does not fit) and RS_LAUNCH_PDL (programmatic dependent
 * launch: may start while the previous kernel in the stream drains). */
#define RS_LAUNCH_COOPERATIVE 1u
#define RS_LAUNCH_PDL 2u
int rs_launch_ex(rs_function f, const unsigned grid[3], const unsigned block[3],
                 const unsigned cluster[3], unsigned smem, void* stream, void** args, unsigned flags);

/* ---- memory (replaces cexec.flatten_value/unflatten_value, cexec.py:533-552) */

int rs_malloc(void** dptr, size_t bytes);
int rs_free(void* dptr);
int rs_memcpy_htod(void* dst, const void* src, size_t bytes, void* stream);
int rs_memcpy_dtoh(void* dst, const void* src, size_t bytes, void* stream);
int rs_memcpy_dtod(void* dst, const void* src, size_t bytes, void* stream);
int rs_memset_d8(void* dst, unsigned char value, size_t bytes, void* stream);
/* Device-to-device copy between two GPUs of this node (cuMemcpyPeerAsync
 * over NVLink / NVSwitch; SURVEY.md §8 b "rs_memcpy_...peer"): dst on
 * dst_device, src on src_device, ordered on `stream` of the calling
 * process's device.  src_device == dst_device is a plain device copy. */
int rs_memcpy_peer(void* dst, int dst_device, const void* src, int src_device, size_t bytes, void* stream);

/* ---- streams / events ------------------------------------------------ */

int rs_stream_create(void** stream);
int rs_stream_destroy(void* stream);
int rs_stream_synchronize(void* stream);
int rs_device_synchronize(void);
int rs_event_create(void** event);
int rs_event_destroy(void* event);
int rs_event_record(void* event, void* stream);
int rs_event_synchronize(void* event);
int rs_event_elapsed_ms(float* ms, void* start, void* end);
/* Work enqueued on `stream` after this call waits for `event`'s last record
 * (cross-stream ordering without a host sync; Executable uses it to keep an
 * executable's stateful workspaces — launch counters, exchange slots — in
 * launch order when one executable is launched on several streams). */
int rs_stream_wait_event(void* stream, void* event);

/* ---- CUDA graphs (launch-bound multi-kernel steps) --------------------
 * Capture everything enqueued on `stream` between begin and end (e.g. every
 * stage of a multi-kernel unit, bound once) into an executable graph, then
 * replay it with one launch.  Replaces: nothing (cexec interprets text). */
int rs_graph_capture_begin(void* stream);
int rs_graph_capture_end(void* stream, void** graph_exec);
int rs_graph_launch(void* graph_exec, void* stream);
/* Upload the graph's work to the device ahead of its first launch (the
 * first launch then pays no upload: cuGraphUpload). */
int rs_graph_upload(void* graph_exec, void* stream);
int rs_graph_destroy(void* graph_exec);

/* ---- TMA ------------------------------------------------------------- */

/* Encode a 2-D (inner dim0, outer dim1) tiled TMA descriptor for fp32 data
 * into the 128-byte buffer `desc` (CUtensorMap layout).  `row_stride_bytes`
 * is the byte distance between consecutive dim1 rows (multiple of 16).
 * `swizzle`: 0 none, 1 32B, 2 64B, 3 128B, 4 128B with 32-byte atoms (the
 * layout tcgen05 reads MN-major tf32 operands in).  Out-of-bounds box elements are
 * zero-filled by the hardware. */
int rs_tma_desc_2d_f32(void* desc, const void* base,
                       uint64_t dim0, uint64_t dim1, uint64_t row_stride_bytes,
                       uint32_t box0, uint32_t box1, int swizzle);

/* ---- multi-GPU: peer memory and collectives (SURVEY.md §8 e) --------
 * The reference runs on one (sequentialised) device; nothing is replaced.
 * One process per GPU.  Out-of-band exchange of the opaque handles / ids
 * below is the caller's plumbing (torch.distributed in the Python side). */

/* Cross-process peer memory over NVLink: export the allocation holding
 * `dptr` as a 64-byte CUDA IPC handle plus the byte offset of `dptr` in it. */
int rs_ipc_handle(void* handle_out /* 64 bytes */, size_t* offset_out, const void* dptr);
/* Map a peer's exported allocation into this process (peer access enabled
 * lazily); *dptr_out = mapped base + offset.  Same-process handles fail. */
int rs_ipc_open(void** dptr_out, const void* handle /* 64 bytes */, size_t offset);
/* Unmap a pointer returned by rs_ipc_open. */
int rs_ipc_close(void* dptr);

/* Halo exchange of a row band laid out [rows + 2][row_bytes]: rows 1..rows
 * are this rank's; row 0 receives the LAST owned row of the band above
 * (`above`, its band base as mapped by rs_ipc_open, holding `above_rows`
 * owned rows) and row rows+1 the FIRST owned row of the band below
 * (`below`).  A NULL neighbour is a global edge: the halo row is the clamped
 * copy of the band's own edge row (padClamp2D semantics, the halo rows of
 * shard.halo_exchange_rows).  Enqueued on `stream` as device-to-device
 * copies (NVLink for peers); the caller orders them after the neighbours'
 * producers (e.g. a barrier) — a pull model, no send side. */
int rs_halo_exchange(void* band, size_t row_bytes, size_t rows, const void* above, size_t above_rows,
                     const void* below, void* stream);

/* NCCL communicator (libnccl.so.2 is loaded at run time). */
typedef struct rs_comm_s* rs_comm;
/* A fresh 128-byte ncclUniqueId (rank 0 creates it, every rank passes it). */
int rs_comm_unique_id(void* id_out /* 128 bytes */);
int rs_comm_init(rs_comm* out, int nranks, int rank, const void* id /* 128 bytes */);
int rs_comm_destroy(rs_comm comm);
/* recv[r * bytes_per_rank ...] = rank r's send buffer, for every rank r, in
 * rank order (the dot partials and the nbody positions of shard.py). */
int rs_allgather(rs_comm comm, const void* send, void* recv, size_t bytes_per_rank, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RISE_B200_H */
