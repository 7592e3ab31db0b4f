/*
 * hetjpeg_b200.h - C ABI of the B200-native "parallel phase" of the hetjpeg
 * JPEG decoder (dequantise -> IDCT -> chroma upsample -> YCbCr->RGB) and of
 * its host entropy stage.
 *
 * Plain pointers and sizes only; no CUDA or torch types.  Every function
 * returns an hj_status (0 = OK); hj_last_error() gives the message of the
 * calling thread's last failure.  Streams are passed as `void*` holding a
 * cudaStream_t (NULL = the library's per-thread default stream).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference root, pkg/src/hetjpeg/...).
 */
#ifndef HETJPEG_B200_H
#define HETJPEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  1..4 mirror the native decoder's ERR_* enum
 * (kernels/_native.pyx:18-23); the host wrapper maps them onto the
 * reference exception classes (errors.py:4-69). */
typedef enum {
    HJ_OK = 0,
    HJ_ERR_EXHAUSTED = 1,   /* BitstreamExhausted */
    HJ_ERR_BADCODE = 2,     /* BadCode */
    HJ_ERR_MARKER = 3,      /* MarkerInScan (non-restart marker) */
    HJ_ERR_RST_SEQ = 4,     /* MarkerInScan (restart out of sequence) */
    HJ_ERR_ARG = 16,        /* invalid argument (ValueError) */
    HJ_ERR_CUDA = 17,       /* CUDA runtime failure */
    HJ_ERR_NOMEM = 18,      /* allocation failure */
    HJ_ERR_NODEVICE = 19    /* no CUDA device visible */
} hj_status;

/* Chroma subsampling of a frame.  420 is this library's documented
 * extension: the reference accepts only 4:4:4 and 4:2:2
 * (parser.py:223-229); see DESIGN.md "4:2:0 extension". */
enum { HJ_SUB_444 = 0, HJ_SUB_422 = 1, HJ_SUB_420 = 2 };

/* Flags for hj_image_t.flags */
enum {
    HJ_FLAG_DIRECT_IDCT = 1,  /* idct="direct" (cli.py:249); default AAN "fast" */
    HJ_FLAG_ISLOW_IDCT = 2    /* idct="islow": libjpeg's integer decode (jidctint islow IDCT,
                                 jdsample fancy upsampling with real-size edges, jdcolor
                                 colour) - north_star's fixed-point mode; not the
                                 reference's float64 arithmetic */
};
/* The `fast` argument of hj_render_rows: the IDCT path. */
enum { HJ_IDCT_DIRECT = 0, HJ_IDCT_FAST = 1, HJ_IDCT_ISLOW = 2 };

/* One image (or an MCU-row range of one) for the device-resident batch API.
 * All pointers are DEVICE pointers.  Layout of the coefficient planes is the
 * reference CoefficientBuffer (entropy.py:31-56): int16 [n_blocks][64],
 * natural (de-zigzagged) order, Y blocks MCU-ordered (ypm = 1/2/4 per MCU).
 * q is the (3,64) int32 de-zigzagged qtable stack (perf_model.py:306-311).
 * rgb is (height, width, 3) uint8, row-major (block_transforms.py:45-57). */
typedef struct {
    const int16_t *y;
    const int16_t *cb;
    const int16_t *cr;
    const int32_t *q;
    uint8_t *rgb;
    int32_t width, height;
    int32_t mcus_per_row, mcu_rows;
    int32_t row0, n_rows;   /* MCU rows to render: [row0, row0+n_rows) */
    int32_t subsampling;    /* HJ_SUB_* */
    int32_t flags;          /* HJ_FLAG_* */
} hj_image_t;

/* ---- library / device ------------------------------------------------ */
const char *hj_version(void);
const char *hj_last_error(void);
int hj_device_count(void);
hj_status hj_set_device(int device);

/* Device / pinned-host memory and copies, so hosts need no other CUDA binding. */
hj_status hj_malloc_device(void **ptr, size_t bytes);
hj_status hj_free_device(void *ptr);
hj_status hj_malloc_host(void **ptr, size_t bytes);     /* page-locked */
hj_status hj_free_host(void *ptr);
hj_status hj_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream);
hj_status hj_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream);
hj_status hj_memset_device(void *dst, int value, size_t bytes, void *stream);
hj_status hj_stream_create(void **stream);
hj_status hj_stream_destroy(void *stream);
hj_status hj_stream_synchronize(void *stream);
hj_status hj_device_synchronize(void);

/* Events for device-side timing on a given stream. */
hj_status hj_event_create(void **event);
hj_status hj_event_destroy(void *event);
hj_status hj_event_record(void *event, void *stream);
hj_status hj_event_elapsed_ms(void *start, void *end, float *ms);
/* Make `stream` wait (on the device) for `event` (cross-stream pipelining). */
hj_status hj_stream_wait_event(void *stream, void *event);

/* ---- the parallel phase: device-resident batch ---------------------- */
/* Render every image of the batch on `stream` (asynchronous).  Replaces the
 * per-lane render_rows dispatch (block_transforms.py:60-75 ->
 * kernels/_native.pyx:493-549) with one launch per subsampling present.
 * Output rows [8*row0*vs, min(h, 8*vs*(row0+n_rows))) are written (vs = 2 for
 * 4:2:0, else 1); nothing else.  4:2:0 reads the chroma blocks of MCU rows
 * row0-1 and row0+n_rows when they exist (the vertical filter's context). */
hj_status hj_render_batch(const hj_image_t *images, int n_images, void *stream);

/* Reusable launch plan for a fixed batch (tile list resident on the device;
 * what a CUDA graph or a steady-state pipeline replays).  The hj_image_t
 * array is copied at creation: pointers inside it must stay valid. */
hj_status hj_plan_create(const hj_image_t *images, int n_images, void **plan);
hj_status hj_plan_launch(void *plan, void *stream);
hj_status hj_plan_destroy(void *plan);

/* Number of kernel launches hj_render_batch issued since library load
 * (evidence for the bench's gpu_launches claim). */
uint64_t hj_launch_count(void);

/* Blocks the render kernel's binary32 screen could not prove and recomputed
 * in exact float64 (cumulative, all launches). */
uint64_t hj_exact_block_count(void);

/* Launches of the tensor-core IDCT-screen kernel (opt-in with HJ_RENDER_TC=1 in
 * the environment), cumulative since library load. */
uint64_t hj_tc_launch_count(void);

/* Packed coefficient transfer of the synchronous drop-in (hj_render_rows*):
 * the host packs each block into a 64-bit nonzero mask of its AC coefficients,
 * a 32-bit value offset (bit 31: int16 values), its int16 DC and its nonzero AC
 * coefficients (int8 when all fit), copies that, and expands it on the device -
 * lossless; the copy is PCIe-bound and 1080p q90 blocks shrink from 128 to
 * ~47 B.  Default (mode -1): packed when the host CPU has AVX-512 VBMI2, >= 4
 * calls are in flight (a saturated link) and the call's first 4096 Y blocks
 * pack below 0.45 of their dense bytes; otherwise dense.  Calls above 64k
 * blocks are packed in bands (hj_set_pack_band).
 * Mode 0 forces the dense copy, 1 forces packing; HJ_PACK_H2D=0/1 in the
 * environment does the same.  hj_packed_h2d_active: 0 off, 1 forced, 2 auto. */
hj_status hj_set_packed_h2d(int32_t mode);
int32_t hj_packed_h2d_active(void);
/* Packed calls above 64k blocks (default) are sent in bands of MCU rows of
 * ~32k blocks: band k+1 packs on the host while band k copies and band k-1
 * renders and returns its RGB rows.  hj_set_pack_band(n > 0) sets both the
 * threshold and the band size to n blocks (tests; HJ_PACK_BAND=n in the
 * environment does the same); 0 restores the default. */
hj_status hj_set_pack_band(int64_t blocks);
/* Bytes the synchronous drop-in copied host->device so far (packed or dense). */
uint64_t hj_h2d_bytes(void);
/* The packer / a host unpacker (tests): returns the value bytes written. `vals`
 * needs 130 * n + 128 bytes. */
int64_t hj_pack_blocks(const int16_t *src, int64_t n, uint64_t *mask, uint32_t *off, int16_t *dc,
                       uint8_t *vals);
hj_status hj_unpack_blocks_host(const uint64_t *mask, const uint32_t *off, const int16_t *dc,
                                const uint8_t *vals, int64_t n, int16_t *dst);

/* ---- the parallel phase: synchronous host-buffer drop-in -------------- */
/* Exactly the backend contract of render_rows_444 / render_rows_422
 * (kernels/_native.pyx:532-549, kernels/fallback.py:224-260): HOST arrays,
 * blocks of the whole image, rgb (height, width, 3) written in place for the
 * MCU rows [row0, row0+n_rows); returns after the RGB rows are in `rgb`.
 * `fast` selects the AAN (1) or direct-basis (0) transform of the
 * reference, or HJ_IDCT_ISLOW (2) for libjpeg's islow decode; `fused` is
 * accepted for interface parity and never changes bytes.  y/cb/cr must hold
 * every block of the image (n_y_blocks / n_c_blocks give their counts, used
 * for bounds checks).  Re-entrant: each host thread uses its own stream and
 * staging buffers. */
hj_status hj_render_rows(const int16_t *y, const int16_t *cb, const int16_t *cr,
                         const int32_t *q3x64, uint8_t *rgb,
                         int32_t width, int32_t height, int32_t mcus_per_row,
                         int32_t mcu_rows, int32_t row0, int32_t n_rows,
                         int32_t subsampling, int32_t fast, int32_t fused,
                         int64_t n_y_blocks, int64_t n_c_blocks);

/* hj_render_rows plus the device time of its three phases, measured with
 * CUDA events on the library's stream: phase_ms[0] = H2D of the coefficient
 * rows (+ plan), [1] = render kernel(s), [2] = D2H of the RGB rows.  This is
 * what the accelerator lane reports where the reference's simulated lane
 * sleeps (executors.py:163-187: write / compute / read). */
hj_status hj_render_rows_timed(const int16_t *y, const int16_t *cb, const int16_t *cr,
                               const int32_t *q3x64, uint8_t *rgb,
                               int32_t width, int32_t height, int32_t mcus_per_row,
                               int32_t mcu_rows, int32_t row0, int32_t n_rows,
                               int32_t subsampling, int32_t fast, int32_t fused,
                               int64_t n_y_blocks, int64_t n_c_blocks, float *phase_ms);

/* Single-block transforms for the reference's per-block API
 * (block_transforms.py / fallback.py:103-119): n dequantised blocks
 * (int32, natural order) -> 64 samples each (uint8, +128, rounded, clamped),
 * or the float64 pre-rounding core.  HOST buffers, synchronous. */
hj_status hj_idct_blocks(const int32_t *deq, int64_t n, uint8_t *out, int32_t fast);
hj_status hj_idct_blocks_f64(const int32_t *deq, int64_t n, double *out, int32_t fast);
/* Algorithm 1 single-row 4:2:2 upsample (fallback.py:122-139):
 * n rows of 8 chroma samples -> 16 int32 each; left/right[i] < 0 means "no
 * neighbour" (end pixel copied).  HOST buffers, synchronous. */
hj_status hj_upsample_422(const uint8_t *rows, const int16_t *left, const int16_t *right,
                          int32_t *out, int64_t n);
/* Colour conversion of n sample triples (fallback.py:142-150). HOST buffers. */
hj_status hj_ycbcr_to_rgb(const uint8_t *y, const uint8_t *cb, const uint8_t *cr,
                          uint8_t *rgb, int64_t n);

/* ---- host entropy stage (CPU, C++) ------------------------------------ */
/* Packed scan tables, the arrays entropy._pack_scan_tables builds
 * (entropy.py:59-84): 8 slots (0-3 DC, 4-7 AC). */
typedef struct {
    uint8_t lut_sym[8][256];
    uint8_t lut_len[8][256];
    int32_t mincode[8][17];
    int32_t maxcode[8][17];
    int32_t valptr[8][17];
    uint8_t symbols[8][256];
    int32_t comp_dc[3];
    int32_t comp_ac[3];
} hj_scan_tables_t;

/* Huffman-decode MCU rows [row0, row0+n_rows) into the coefficient planes
 * (HOST buffers).  Replaces decode_mcu_rows (kernels/_native.pyx:195-305,
 * fallback.py:282-417): identical bit reader, lookahead + maxcode walk,
 * EXTEND, EOB/ZRL, restart handling and int64[8] resumable state
 * {pos, bitbuf, bits, mcus_since_rst, next_rst, predY, predCb, predCr}.
 * On error the state is still written back (native behaviour) and the
 * HJ_ERR_* code returned. */
hj_status hj_decode_mcu_rows(const uint8_t *data, int64_t n_bytes, int64_t *state,
                             const hj_scan_tables_t *scan,
                             int16_t *y_out, int16_t *cb_out, int16_t *cr_out,
                             int32_t row0, int32_t n_rows, int32_t mcus_per_row,
                             int32_t y_per_mcu, int32_t restart_interval);

/* Throughput decoder for whole scans (pipelined / batched decode): same
 * coefficients as hj_decode_mcu_rows, 64-bit bit buffer + 10-bit lookahead
 * with fused run/size/value AC decode, and the scan split at its RSTn markers
 * across up to n_threads host threads (exact: RSTn resets the predictors,
 * kernels/_native.pyx:238-257).  Every block of the planes is written (no
 * pre-zeroing needed).
 * hj_huff_build packs the tables once per scan header. */
hj_status hj_huff_build(const hj_scan_tables_t *scan, void **fast);
void hj_huff_free(void *fast);
hj_status hj_decode_scan_fast(const void *fast, const uint8_t *data, int64_t n_bytes,
                              int16_t *y_out, int16_t *cb_out, int16_t *cr_out,
                              int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu,
                              int32_t restart_interval, int32_t n_threads);

/* MCU rows [row0, row0+n_rows) of a scan: only the restart intervals that
 * cover them are Huffman-decoded (their blocks written, zeros included), on up
 * to n_threads threads - a shard of one large image (BASELINE config 4,
 * MCU-row shards across GPUs) pays only for its own intervals.  Without
 * restart intervals the whole scan is decoded. */
hj_status hj_decode_scan_rows(const void *fast, const uint8_t *data, int64_t n_bytes,
                              int16_t *y_out, int16_t *cb_out, int16_t *cr_out,
                              int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu,
                              int32_t restart_interval, int32_t row0, int32_t n_rows, int32_t n_threads);

/* ---- native batch pipeline (pipeline.BatchDecoder; the paper's pipelined
 * host-Huffman / accelerator scheme, §5.3, at batch granularity).
 * One image: its scan (hj_huff_build tables + entropy-coded bytes), its
 * page-locked host coefficient planes and RGB, its device planes / RGB and
 * an hj_plan_create plan rendering it from those device planes. */
typedef struct {
    const void *huff;
    const uint8_t *scan;
    int64_t scan_bytes;
    int16_t *y, *cb, *cr;                 /* host planes (page-locked) */
    void *dev_y, *dev_cb, *dev_cr;        /* device planes */
    int64_t n_y, n_c;                     /* blocks in the Y / each chroma plane */
    int32_t mcus_per_row, mcu_rows, y_per_mcu, restart_interval;
    void *plan;
    const void *dev_rgb;
    uint8_t *rgb;                         /* host RGB (page-locked) */
    int64_t rgb_bytes;
} hj_pipe_image_t;

/* n_threads host threads each take the next image, entropy-decode it
 * (hj_decode_scan_fast) and queue its H2D -> render -> D2H on streams[t];
 * returns once every stream has drained (first error wins). */
hj_status hj_pipeline_run(const hj_pipe_image_t *images, int32_t n_images, int32_t n_threads,
                          void *const *streams);
/* The same host stage alone (T_huff of the Amdahl bound, orchestrator.py:71-75). */
hj_status hj_pipeline_huffman(const hj_pipe_image_t *images, int32_t n_images, int32_t n_threads);

/* ---- host/accelerator row split (partitioner, Eq. 10-15) -----
 * A balance f(x) = sum_i sign_i * P_i(a_i), P_i an ascending univariate
 * polynomial (the DeviceProfile's models restricted to the image width; a
 * constant is a 1-coefficient polynomial) and a_i = x (host rows) or h - x
 * (accelerator rows, `reflected`).  hj_partition_solve finds its root on
 * [0, h] (Newton on the analytic derivative, bisection fallback; the
 * iteration limits and tolerances of partitioner.py:95-135) and rounds the
 * accelerator share to whole MCU rows from the top (partitioner.py:138-155).
 * Replaces partitioner._solve_balance / _to_plan. */
typedef struct {
    const double *coef;
    int32_t n;          /* coefficients, ascending powers */
    int32_t reflected;  /* evaluate at h - x */
    double sign;        /* +1 or -1 */
} hj_balance_term_t;

typedef struct {
    double x_root;                      /* host rows before rounding */
    int32_t accel_mcu_rows, cpu_mcu_rows;
    int32_t accel_rows, cpu_rows;       /* pixel rows */
} hj_partition_t;

hj_status hj_partition_solve(const hj_balance_term_t *terms, int32_t n_terms, int32_t h, int32_t mcu_height,
                             hj_partition_t *out);
/* f(x) (and f'(x) in *slope when non-NULL) of a balance - tests and diagnostics. */
double hj_balance_eval(const hj_balance_term_t *terms, int32_t n_terms, double h, double x, double *slope);

/* ---- streaming decode with a bounded ring (BASELINE config 5) ---------
 * One image of a stream: its scan (hj_huff_build tables + entropy-coded
 * bytes), its host qtables and its geometry.  rgb_out: host destination of
 * its RGB (page-locked for an asynchronous copy), or NULL to leave it in the
 * ring's own page-locked slot (delivered and then overwritten). */
typedef struct {
    const void *huff;
    const uint8_t *scan;
    int64_t scan_bytes;
    const int32_t *q;                     /* (3, 64) host qtables */
    int32_t width, height, subsampling;   /* HJ_SUB_* */
    int32_t flags;                        /* HJ_FLAG_* (IDCT path) */
    int32_t restart_interval;
    uint8_t *rgb_out;
    int32_t row0, n_rows;                 /* MCU rows to decode and render (n_rows 0 = all): an
                                             image shard - only its restart intervals are
                                             Huffman-decoded (4:2:0: plus one chroma MCU row of
                                             context each side) and only its RGB rows move */
} hj_stream_image_t;

typedef struct {
    int64_t images, launches;
    int64_t h2d_bytes, d2h_bytes;         /* moved by the GPU leg */
    int64_t pinned_bytes, device_bytes;   /* the ring's whole footprint */
    double huffman_thread_s;              /* summed host entropy-decode time */
    double wall_s;                        /* first image taken -> last RGB delivered (ring set-up excluded) */
} hj_stream_stats_t;

/* Decode n images in list order with n_slots reusable slots (page-locked
 * planes + device planes + stream each, sized to the largest image): n_threads
 * host threads Huffman-decode into free slots; the calling thread queues each
 * decoded slot's H2D -> render -> D2H and recycles finished slots.  Memory is
 * bounded by the slots, not the list.  gpu = 0: the host stage alone (T_huff).
 * Replaces the reference's per-image decode loop (cli.py:175-234) for a
 * whole corpus; first error wins. */
hj_status hj_stream_run(const hj_stream_image_t *images, int32_t n, int32_t n_threads, int32_t n_slots,
                        int32_t gpu, hj_stream_stats_t *stats);

/* Index of the first non-restart marker after the scan data starting at
 * `start`, or -1 if the stream ends inside the entropy-coded data
 * (parser.py:277-293, _scan_entropy_end). */
int64_t hj_scan_entropy_end(const uint8_t *data, int64_t n_bytes, int64_t start);

#ifdef __cplusplus
}
#endif

#endif /* HETJPEG_B200_H */
