/* emt_b200.h — C ABI of the B200 EMT step-loop engine (libemtb200.so).
 *
 * Drop-in for the reference executor boundary:
 *
 *   WaveformSet interpret(const ScheduleProgram&, const Eigen::VectorXd& initial,
 *                         int steps, const ExecOptions& = {});
 *     /root/reference/proj/include/emtgrid/exec.hpp:29-30, proj/src/exec.cpp:350-383
 *   WaveformSet execute_parallel(const ScheduleProgram&, const Eigen::VectorXd&, int workers,
 *                                int steps, const ExecOptions& = {});
 *     /root/reference/proj/include/emtgrid/exec.hpp:36-37, proj/src/exec.cpp:385-500
 *   dispatched from execute_task, proj/src/pipeline.cpp:20-33
 *
 * The schedule crosses the boundary in the reference's own canonical text
 * form (ScheduleProgram::serialize, proj/src/schedule.cpp:335-411; grammar in
 * proj/docs/schedule_format.md). The initial arena is `extent*width` doubles,
 * slot-major with lanes innermost (proj/docs/schedule_format.md:32-34), exactly
 * the reference's Eigen::VectorXd. Waveforms come back in WaveformSet order:
 * `steps` rows of `channels*width` doubles, column = channel*width + lane
 * (proj/include/emtgrid/waveform.hpp:12-37).
 *
 * Plain pointers and sizes only. Every call is synchronous unless it says
 * otherwise. An engine is confined to one host thread at a time.
 */
#ifndef EMT_B200_H
#define EMT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status = 0 on success, else 1 + emtgrid::ErrorCode
 * (proj/include/emtgrid/common.hpp:11-33), plus engine-specific codes >= 64. */
typedef enum emt_status {
    EMT_OK = 0,
    EMT_MALFORMED_DOCUMENT = 1,
    EMT_NON_FINITE_STATE = 7,   /* |v| > divergence limit, proj/src/exec.cpp:229-237 */
    EMT_SINGULAR_MATRIX = 8,    /* pivot check, proj/src/sparse.cpp:135-143 */
    EMT_DIMENSION_MISMATCH = 10,/* initial.size() != extent*width, proj/src/exec.cpp:340-346 */
    EMT_TOPOLOGY_MISMATCH = 12, /* batch not isomorphic to the compiled one (cf. vectorize, proj/src/cgm.cpp:367) */
    EMT_CAPACITY_EXCEEDED = 13, /* arena does not fit the device plan */
    EMT_UNKNOWN_KIND = 14,      /* unregistered kernel code, proj/src/exec.cpp:37-41 */
    EMT_NON_POSITIVE_INPUT = 20,/* steps < 0, width < 1, ... */
    EMT_CUDA_ERROR = 64,        /* CUDA runtime failure (message has the detail) */
    EMT_INVALID_HANDLE = 65,
    EMT_INEXACT_DIVISION = 66,  /* a nonzero backward-sweep quotient fell below 2^-900, where the
                                   fast reciprocal division may misround: rerun the batch with
                                   EMT_FLAG_EXACT_DIVISION (emt_interpret does this itself) */
} emt_status;

typedef struct emt_engine emt_engine;

/* Where and how an engine runs. Zero-initialise for defaults. */
typedef struct emt_config {
    int32_t device;          /* CUDA device ordinal */
    int32_t lane_begin;      /* first scenario lane this engine owns (multi-GPU shard) */
    int32_t lane_count;      /* lanes owned; 0 = all lanes from lane_begin */
    int32_t lanes_per_block; /* generic kernel: warps (= lanes) per CTA, 0 = auto */
    int32_t warps_per_group; /* specialised kernel: warps sharing one 32-lane group, 0 = auto (8) */
    int32_t kernel;          /* EMT_KERNEL_AUTO / _SPECIALISED / _GENERIC / _TSIMT */
    int32_t flags;           /* EMT_FLAG_* */
    int32_t reserved;
} emt_config;

/* Shared-G batches (no switches; every conductance a lane-invariant constant):
 * replace the sparse forward/backward sweeps by V = G^-1 I on the FP64 tensor
 * cores (mma.sync m8n8k4, specialised kernel). Reassociates the solve: results
 * agree to ~1e-15 of the signal amplitude, not bit-for-bit.
 * Ignored (exact LU solve) when the batch is not shared-G. */
enum { EMT_FLAG_TENSOR_SOLVE = 1 };

/* The specialised kernel divides by a pivot as q = x*r, x/u = fma(fma(-u, q, x), r, q)
 * with r = 1/u (Markstein: the IEEE quotient bit for bit while q is zero or
 * |q| >= 2^-900 and |u| is in [2^-60, 2^960]). By default each backward row only
 * checks that bound (one compare, no branch) and a pass that breaks it stops the
 * launch with EMT_INEXACT_DIVISION; with this flag every row branches to IEEE
 * x / u below the bound instead (exact everywhere, ~20% slower). */
enum { EMT_FLAG_EXACT_DIVISION = 2 };

/* Cold start: engine creation returns at once and the engine runs the generic
 * kernel (bit-identical) while the specialised kernel is generated and
 * NVRTC-compiled on a host thread; the first launch after the compile finishes
 * switches to it. AUTO kernel selection only; ignored for line-coupled batches,
 * the tensor-core solve and lanes too large for the generic kernel's shared
 * memory. emt_engine_wait_jit() blocks until the switch. */
enum { EMT_FLAG_ASYNC_JIT = 4 };

/* Step-loop kernel selection. AUTO generates and JIT-compiles (NVRTC) a kernel
 * specialised to the schedule — the code generator of the reference's
 * emit_source (proj/src/codegen.cpp:84-230) retargeted to sm_100a — and uses
 * the table-driven generic kernel only when the specialised one cannot be
 * built (e.g. the hot arena exceeds shared memory). Both run on the GPU. */
enum { EMT_KERNEL_AUTO = 0, EMT_KERNEL_SPECIALISED = 1, EMT_KERNEL_GENERIC = 2, EMT_KERNEL_TSIMT = 3, EMT_KERNEL_SYSTEM = 4 };
/* EMT_KERNEL_SYSTEM: one 1024-thread CTA per lane for large single systems (the
 * reference's gen_scale_case, proj/src/bench.cpp:54-117): the arena stays in HBM,
 * layers run in parallel over the block, the forward sweep in 32-column blocks and
 * the backward sweep streams U through a TMA ring. AUTO selects it when a lane's
 * arena does not fit in shared memory. Bit-identical to the other kernels. */
/* EMT_KERNEL_TSIMT: generated task-SIMT kernel — one CTA per scenario lane, one
 * thread per task of a DAG wave (codegen.cpp, generate_tsimt); for few lanes
 * (latency) and for batches that should spread over every SM. */

/* ExecOptions (proj/include/emtgrid/exec.hpp:17-25). */
typedef struct emt_exec_options {
    double divergence_limit; /* <= 0 selects kDivergenceLimit = 1e12 (kernels.hpp:24) */
    int32_t warmup_steps;    /* steps excluded from measured_seconds */
    int32_t reserved;
} emt_exec_options;

/* ExecStats (proj/include/emtgrid/exec.hpp:10-15) plus device counters. */
typedef struct emt_exec_stats {
    int32_t factor_count;    /* refactorization passes; == reference lane-0 fcount */
    int32_t measured_steps;
    double measured_seconds; /* device time of the step loop after warm-up (CUDA events) */
    int32_t kernel_launches; /* kernels launched (step loop + per-launch source tables) */
    int32_t switch_events;   /* (step, lane, switch) state changes seen */
} emt_exec_stats;

/* One switch state change: the process id of the switch's Norton update
 * (== its canonical component index) changed state at `step` in `lane`. */
typedef struct emt_switch_event {
    int32_t step;
    int32_t lane;
    int32_t process;
} emt_switch_event;

/* ---- one-shot drop-in for interpret() ------------------------------------ */

/* Parses `schedule_text`, runs `steps` passes from `initial` on `cfg->device`
 * and writes the waveform rows. `waves` holds steps*channels*width doubles
 * (may be NULL), `time` holds `steps` doubles (may be NULL). On error the
 * status mirrors the reference exception and emt_last_error() carries
 * "<where>: <message>". */
emt_status emt_interpret(const char* schedule_text, const double* initial, int64_t initial_len,
                         int32_t steps, const emt_exec_options* options, const emt_config* cfg,
                         double* waves, double* time, emt_exec_stats* stats);

/* ---- multi-device executor (SURVEY §8(b) emt_create / emt_run) ----------- */

/* One engine over `ndev` devices: the batch's `width` lanes are split into
 * contiguous shards, one lane-shard engine per listed device (a device may be
 * listed twice), all run concurrently from the calling thread. `initial` holds
 * extent*width doubles (the reference arena); the schedule text carries the
 * batch's constant table. The engine is confined to one host thread at a time. */
typedef struct emt_multi emt_multi;
typedef emt_exec_stats emt_stats;
emt_status emt_create(const char* cgmsched_text, const double* initial, int64_t extent, int32_t width,
                      const int32_t* devices, int32_t ndev, emt_multi** out);
/* `steps` passes from the initial arena (`warmup` of them outside measured_seconds);
 * waves: steps x (channels * width), the WaveformSet row layout (may be NULL).
 * factor_count counts a pass once when any lane refactorises (exec.cpp:200-201);
 * measured_seconds is the slowest device's. On error the lowest-lane shard that
 * failed reports. */
emt_status emt_run(emt_multi* engine, int32_t steps, int32_t warmup, double* waves, emt_stats* out);
/* "<where>: <message>" of the engine's last failing call. */
const char* emt_error_detail(const emt_multi* engine);
void emt_destroy(emt_multi* engine);

/* Twin of execute_parallel (proj/include/emtgrid/exec.hpp:35-37): the same
 * results as emt_interpret; workers < 1 fails with NonPositiveInput as there. */
emt_status emt_execute_parallel(const char* schedule_text, const double* initial, int64_t initial_len,
                                int32_t workers, int32_t steps, const emt_exec_options* options,
                                const emt_config* cfg, double* waves, double* time, emt_exec_stats* stats);

/* Thread-local detail of the last failing call on this thread. */
const char* emt_last_error(void);

/* ---- engine object: resident batch, resumable stepping -------------------- */

/* `const_table` (optional, may be NULL): consts*width doubles, slot-major,
 * replacing the CONST rows of the text (lets callers widen a base schedule to
 * `width` scenario lanes without re-serialising it); `width` must then be
 * given, else it is read from the schedule header. */
emt_status emt_engine_create(const char* schedule_text, const double* const_table, int32_t width,
                             const double* initial, int64_t initial_len, const emt_config* cfg,
                             emt_engine** out);
void emt_engine_destroy(emt_engine* engine);

/* Shape: lanes owned by this engine, channels, arena extent, const extent,
 * META steps, nodes, L nnz, U nnz, layers. Any pointer may be NULL. */
emt_status emt_engine_shape(const emt_engine* engine, int32_t* lanes, int32_t* channels,
                            int32_t* extent, int32_t* consts, int32_t* steps, int32_t* nodes,
                            int32_t* l_nnz, int32_t* u_nnz, int32_t* layers);

/* Reserves device waveform storage for `capacity_steps` recorded passes and
 * rewinds the recorder. Called implicitly by emt_engine_run. */
emt_status emt_engine_reserve(emt_engine* engine, int32_t capacity_steps);

/* Advances the device-resident batch by `steps` passes starting at absolute
 * pass index engine->step (t = (step+1)*dt, proj/src/exec.cpp:366), appending
 * waveform rows to device storage. Asynchronous on the engine's stream when
 * `sync` is 0; errors raised inside the kernel surface on the next
 * synchronising call (emt_engine_sync / read / stats). */
emt_status emt_engine_advance(emt_engine* engine, int32_t steps, int32_t sync);
emt_status emt_engine_sync(emt_engine* engine);

/* Reloads the resident batch from host buffers (H2D on the engine's stream,
 * asynchronous w.r.t. the host when the buffers are pinned) and rewinds it to
 * pass 0: `initial` is the whole batch's arena (extent*width doubles, the
 * width the engine was created with; this engine copies its lane slice) and
 * `const_table` (may be NULL = keep) its consts*width constant table. This is
 * the per-job input of interpret() (proj/src/exec.cpp:358 copies `initial`)
 * without re-running the code generator. A const table whose lane-invariant
 * slots differ from the ones the specialised kernel compiled in is rejected
 * with EMT_TOPOLOGY_MISMATCH (create a new engine for it). */
emt_status emt_engine_load(emt_engine* engine, const double* initial, int64_t initial_len,
                           const double* const_table);

/* emt_engine_load in two halves, for pipelining batches: `stage` starts the
 * H2D of the next batch into device staging buffers on a separate stream
 * (returns at once for pinned buffers; it may overlap a running batch), and
 * `commit` makes the staged batch current (the staging and live buffers swap
 * roles, no copy; launches issued after it read the new batch, and the next
 * `stage` writes the old buffers only after every launch issued before the
 * commit has finished) and rewinds to pass 0. */
emt_status emt_engine_stage(emt_engine* engine, const double* initial, int64_t initial_len,
                            const double* const_table);
emt_status emt_engine_commit(emt_engine* engine);

/* Runs `steps` passes in launches of `chunk` passes (<= 0: auto) and, when
 * `waves` is not NULL, streams each finished chunk's rows to `waves`
 * (steps*channels*lanes doubles, WaveformSet layout of this engine's lanes)
 * on a copy stream while the next chunk computes. Returns after the last row
 * has landed; errors as emt_engine_sync. Grows the waveform store as needed
 * (SURVEY.md §8(b) emt_run). */
emt_status emt_engine_run(emt_engine* engine, int32_t steps, int32_t chunk, double* waves);
/* emt_engine_run without the final wait: returns once every launch and copy is
 * enqueued (the host buffer must stay alive and untouched until emt_engine_wait,
 * and the engine must not be reloaded before it). Lets a caller overlap one
 * batch's last waveform copies with the next batch's compute on another engine. */
emt_status emt_engine_run_async(emt_engine* engine, int32_t steps, int32_t chunk, double* waves);
emt_status emt_engine_wait(emt_engine* engine);

/* Line-end history mirror (Bergeron extension, kernel code 20): a device array
 * of `lanes` (= the whole batch width) x `cols` doubles, lane-major, holding
 * every lane's ring slots [ring_lo, ring_lo+cols). Each launch writes this
 * engine's lanes' rows and reads peer rows; an engine that owns a lane shard
 * gets the other shards' rows from its peers between launches (the exchange
 * of a line-split system over several GPUs). `max_chunk` = passes per launch
 * (K-1 of the shortest line), 0 when unbounded. */
emt_status emt_engine_ring(emt_engine* engine, void** device_ptr, int32_t* lanes, int32_t* cols,
                           int32_t* max_chunk);
/* Moves the mirror into caller-owned device memory (lanes*cols doubles, e.g. a
 * buffer a collective library writes into); the engine copies its current
 * contents there and uses it from then on. The buffer must outlive the engine. */
emt_status emt_engine_attach_ring(emt_engine* engine, void* device_ptr);

/* Phase profiler of the specialised kernel (engine created with the
 * environment variable EMTB200_CG_PROF=1): cycles summed over the passes run
 * so far, CTA 0, per warp (32) x marker (64), marker 2p = phase p's compute,
 * 2p+1 = the barrier wait after it, numbered region by region. */
emt_status emt_engine_profile(emt_engine* engine, int64_t* cycles, int32_t n);

/* Device-side exchange for a line-split system over several engines / GPUs:
 * every engine of the system attaches the SAME mirror (lanes x cols doubles,
 * lane-major, see emt_engine_ring) and the SAME progress array (total_ctas
 * uint32), this engine's CTAs being [cta_offset, cta_offset + emt_engine_ctas()).
 * Each engine then runs its launches persistently: its CTAs write their
 * line-end histories straight into the shared mirror and wait on every CTA's
 * progress word (K-1 passes of slack), so no host exchange is needed. With
 * system_scope != 0 the acquire/release and ring reads are system-scoped, for
 * peers on other GPUs (memory from emt_ipc_alloc / emt_ipc_open over NVLink).
 * All engines' launches must be resident together. */
emt_status emt_engine_attach_lines(emt_engine* engine, void* mirror, void* progress, int32_t cta_offset,
                                   int32_t total_ctas, int32_t system_scope);

/* Lane groups of this engine (one CTA each; with the full-chip launch of the
 * specialised kernel the group of SM s runs on SM s and the other CTAs exit) and
 * lanes per group (0 for the generic kernel): the progress-array span
 * emt_engine_attach_lines expects from this engine. */
emt_status emt_engine_ctas(const emt_engine* engine, int32_t* ctas, int32_t* lanes_per_cta);
/* CUDA IPC helpers for the shared mirror / progress arrays: `handle` is 64 bytes. */
emt_status emt_ipc_alloc(int32_t device, int64_t bytes, void** ptr, void* handle);
emt_status emt_ipc_open(int32_t device, const void* handle, void** ptr);
emt_status emt_ipc_close(void* ptr);
emt_status emt_ipc_free(void* ptr);

/* Host copies of recorded rows [row0, row0+rows) (WaveformSet layout, this
 * engine's lanes only) and their times. */
emt_status emt_engine_read_waves(emt_engine* engine, int32_t row0, int32_t rows, double* waves,
                                 double* time);
/* Current arena (extent*lanes doubles, slot-major) — a STATE v1 snapshot body. */
emt_status emt_engine_read_state(emt_engine* engine, double* arena);
/* Recorded switch events so far (up to max); returns total in *count. */
emt_status emt_engine_read_events(emt_engine* engine, emt_switch_event* events, int32_t max,
                                  int32_t* count);
emt_status emt_engine_stats(emt_engine* engine, emt_exec_stats* stats);
/* Absolute pass indices at which some lane of this engine refactorised (up to
 * max; total in *count). The union over shards is a sharded run's factor_count. */
emt_status emt_engine_read_refactor_steps(emt_engine* engine, int32_t* steps, int32_t max, int32_t* count);

/* Raw device pointer of the waveform store (rows x channels x lanes doubles)
 * and the CUDA stream the engine launches on (cudaStream_t as void*). */
void* emt_engine_device_waves(emt_engine* engine);
void* emt_engine_stream(emt_engine* engine);

/* Blocks until an asynchronous JIT (EMT_FLAG_ASYNC_JIT) has finished and adopts its
 * kernel for the following launches; a no-op otherwise. */
emt_status emt_engine_wait_jit(emt_engine* engine);

/* Which kernel the engine runs (EMT_KERNEL_SPECIALISED or _GENERIC), the
 * generated CUDA source (empty for the generic kernel) and a one-line plan
 * summary (tasks, phases, shared-memory bytes, JIT time). */
int32_t emt_engine_kernel(const emt_engine* engine);
const char* emt_engine_source(const emt_engine* engine);
const char* emt_engine_summary(const emt_engine* engine);

/* Generates the specialised kernel source (warps < 0: the task-SIMT kernel
 * with -warps warps) for a schedule without touching a
 * device and, when `compile` != 0, compiles it with NVRTC for `arch`
 * (e.g. "sm_100a"). Returned strings stay valid until the next call on this
 * thread. Used by the build check and the CPU test-suite. */
emt_status emt_codegen(const char* schedule_text, const double* const_table, int32_t width, int32_t warps,
                       int32_t compile, const char* arch, const char** source, const char** summary);

/* ---- the "sm100a" code-database dialect ---------------------------------- */

/* emit_source(schedule, "sm100a") (proj/include/emtgrid/codegen.hpp:28; the
 * reference registers only "cpp", proj/src/codegen.cpp:84-87): a standalone CUDA
 * program for this schedule — its specialised step-loop kernel plus a host main()
 * with the emitted "cpp" program's CLI (--state <file> --steps <n> --out <file>;
 * exit 2 usage/I/O, 3 singular matrix, 4 divergence; proj/data/codedb/cpp/
 * prologue.tpl:87,165,198-224) and the same waveform text, byte for byte. Build
 * with nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false. *source is
 * malloc'd (release with emt_free). Line-coupled schedules: EMT_UNKNOWN_KIND. */
emt_status emt_emit_program(const char* schedule_text, char** source);

/* ---- waveform text (WaveformSet::to_text, proj/src/waveform.cpp:22-42) ---- */

/* Formats `rows` waveform rows as the reference's text form: a header line
 * "time <name>..." (names "<name>#<lane>" when width > 1), then per row the
 * time and channels*width values (channel-major, then lane), each as %.17g
 * (format_g17, proj/src/common.cpp:85-89), space-separated, '\n'-terminated.
 * Byte-identical to the reference; `threads` host threads format row blocks.
 * *out is malloc'd (NUL-terminated, *out_len bytes without the NUL); release
 * it with emt_free. */
emt_status emt_waves_to_text(const char* const* channel_names, int32_t channels, int32_t width,
                             const double* time, const double* values, int64_t rows, int32_t threads,
                             char** out, int64_t* out_len);
void emt_free(void* ptr);

/* ---- source waveform function ---- */

/* y[i] = cos(x[i]) as the device evaluates it for AC sources (kern::source_value,
 * proj/include/emtgrid/kernels.hpp:68-70): glibc's cos, operation for operation
 * (csrc/libmcos.cuh), so bit-identical to the reference's std::cos. Host buffers;
 * for verification of a box's libm against the device. */
emt_status emt_source_cos(int32_t device, const double* x, double* y, int64_t n);

/* Library build string (arch, flags). */
const char* emt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EMT_B200_H */
