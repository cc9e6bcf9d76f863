/*
 * sepconv_b200.h -- C ABI of libsepconv_b200.so, the B200 (sm_100a) implementation
 * of the separable (2r+1)-tap convolution hot path of sepconv_lab
 * (S/ = /root/reference/pkg/src/sepconv_lab/, the reference being arXiv 1711.09791's
 * lab). Plain pointers and sizes only; no torch types.
 *
 * Layout: a stack of `nplanes` float32 planes; element (p, y, x) lives at
 *   base + p*plane_stride + y*row_stride + x        (strides in ELEMENTS)
 * The reference's Image is a list of C-contiguous (rows, cols) planes
 * (S/image.py:26-75); a (P, R, C) buffer is plane_stride = R*C, row_stride = C.
 *
 * All device entry points take DEVICE pointers and a cudaStream_t (as void*),
 * are stream-ordered and asynchronous, validate everything before launching and
 * never allocate or free caller buffers. `sc_two_pass_host_f32` takes HOST
 * pointers and blocks, like the reference's launches (S/executors.py:142-151).
 *
 * Arithmetic is bit-identical to the reference: float32 multiply and add, never
 * fused, folded in the reference order (S/conv.py:1-15).
 */
#ifndef SEPCONV_B200_H
#define SEPCONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python layer maps them onto the reference's exceptions
 * (S/errors.py:4-42). Validation happens before any launch. */
#define SC_OK 0
#define SC_INVALID_ARGUMENT 1  /* InvalidArgumentError: shapes, ranges, aliasing (S/conv.py:68-75) */
#define SC_INVALID_DIMENSION 2 /* InvalidDimensionError: plane smaller than the kernel (S/conv.py:76-79) */
#define SC_UNSUPPORTED_WIDTH 3 /* UnsupportedWidthError: width above 255 (or above 9 on the peer-band and fused-u8 entry points) */
#define SC_CUDA_ERROR 4        /* ExecutionError: a launch or copy failed (S/errors.py:36-42) */
#define SC_NCCL_ERROR 5        /* ExecutionError: NCCL unavailable or a communication call failed */

/* Flags */
#define SC_EXTENDED 0x1  /* row pass over every row: conv_two_pass(extended=True), S/conv.py:417-418 */
#define SC_NO_RING 0x2   /* fused two-pass: leave dst outside the valid region untouched */
#define SC_ZERO_FILL 0x4 /* row pass: dst outside the computed region := 0 (zeroed scratch, S/conv.py:414) */
#define SC_COPY_BACK 0x8 /* single pass: also copy the valid region back into src (S/conv.py:424-449) */

int sc_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char *sc_last_error(void);
/* Number of kernels this library has launched in this process. */
uint64_t sc_launch_count(void);

/* Fused single-read / single-write two-pass, out of place (src and dst must not overlap).
 * dst = the image the reference leaves in `image` after conv_two_pass
 * (S/conv.py:392-421) / convolve_image(TWO_PASS) (S/executors.py:308-326):
 * ring (outside [r,R-r)x[r,C-r)) = src, valid region = V(H0) with H0 zero on rows
 * outside [r,R-r) unless SC_EXTENDED. With SC_NO_RING the dst ring is untouched. */
int sc_two_pass_fused_f32(const float *src, float *dst, int nplanes, int rows, int cols,
                          int64_t src_plane_stride, int64_t dst_plane_stride,
                          int64_t src_row_stride, int64_t dst_row_stride,
                          const float *taps, int width, int flags, void *stream);

/* Row-band form of the fused two-pass for the multi-GPU partitioner: the image is
 * global_rows tall; src holds global rows [src_row0, src_row0+src_rows) (the band
 * plus its r-row halo), dst row 0 is global row dst_row0; output rows
 * [out_lo, out_hi) are produced with the faithful rule and ring in GLOBAL rows. */
int sc_two_pass_band_f32(const float *src, float *dst, int nplanes, int global_rows, int cols,
                         int64_t src_plane_stride, int64_t dst_plane_stride,
                         int64_t src_row_stride, int64_t dst_row_stride,
                         int src_row0, int src_rows, int dst_row0, int out_lo, int out_hi,
                         const float *taps, int width, int flags, void *stream);

/* Same with two disjoint output segments in ONE launch (the band's top and
 * bottom boundary rows after the halo exchange): [out_lo,out_hi) and
 * [out_lo2,out_hi2); either may be empty. */
int sc_two_pass_band2_f32(const float *src, float *dst, int nplanes, int global_rows, int cols,
                          int64_t src_plane_stride, int64_t dst_plane_stride,
                          int64_t src_row_stride, int64_t dst_row_stride,
                          int src_row0, int src_rows, int dst_row0, int out_lo, int out_hi,
                          int out_lo2, int out_hi2, const float *taps, int width, int flags, void *stream);

/* One row band whose halo rows are read straight from the neighbouring bands'
 * buffers (other GPUs' memory mapped with sc_ipc_open; multi-GPU without a
 * separate exchange step). src holds global rows
 * [src_row0, src_row0+src_rows); `above` (may be NULL) holds
 * [above_row0, src_row0), `below` (may be NULL) holds
 * [src_row0+src_rows, below_row0+below_rows). Output rows [out_lo,out_hi) go
 * to dst (row 0 = global row dst_row0). The caller orders the neighbours'
 * writes of those rows before this call (e.g. a stream-ordered barrier). */
int sc_two_pass_band_peer_f32(const float *src, float *dst, int nplanes, int global_rows, int cols,
                              int64_t src_plane_stride, int64_t dst_plane_stride,
                              int64_t src_row_stride, int64_t dst_row_stride, int src_row0, int src_rows,
                              const float *above, int above_row0, int above_rows,
                              int64_t above_plane_stride, int64_t above_row_stride,
                              const float *below, int below_row0, int below_rows,
                              int64_t below_plane_stride, int64_t below_row_stride,
                              int dst_row0, int out_lo, int out_hi, const float *taps, int width, int flags,
                              void *stream);

/* The same band step with device-side readiness signalling between ranks, so a
 * step on FRESH inputs needs no host barrier. sig_self: this band's signal
 * block of 8 u64 words in its own device memory (zero-initialised, exported to
 * the neighbours with sc_ipc_export): [0] ready epoch, [2] / [3] running counts
 * of this band's items that finished reading the band above / below, [4] / [5]
 * how many per launch;
 * sig_above / sig_below: the neighbours' words mapped with sc_ipc_open (NULL at
 * the image edges). epoch: this step's number, 1, 2, ... Every CTA publishes
 * ready = epoch when it starts (the band's inputs are in place, by stream order)
 * and waits for both neighbours' ready >= epoch before its first read or write;
 * every item that read a neighbour's rows counts itself once its copies landed. A neighbour that has started step e has
 * finished step e-1, so ping-pong buffers (step e writes what neighbours read in
 * step e-1) are safe too. sig_err (host-mapped u32, may be NULL) is set when a
 * wait outlives SC_PEER_TIMEOUT_MS (default 20000 ms); the kernel then goes on
 * rather than hang the GPU. Widths up to 9 (the NCCL band plan: up to 31). */
int sc_two_pass_band_peer_sig_f32(const float *src, float *dst, int nplanes, int global_rows, int cols,
                                  int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                                  int64_t dst_row_stride, int src_row0, int src_rows, const float *above,
                                  int above_row0, int above_rows, int64_t above_plane_stride,
                                  int64_t above_row_stride, const float *below, int below_row0, int below_rows,
                                  int64_t below_plane_stride, int64_t below_row_stride, int dst_row0, int out_lo,
                                  int out_hi, const float *taps, int width, int flags, uint64_t *sig_self,
                                  const uint64_t *sig_above, const uint64_t *sig_below, uint64_t epoch,
                                  uint32_t *sig_err, void *stream);

/* Stream-ordered wait until the neighbours reached epoch `value`: word 0 = their
 * launch of it started (ready), word 1 = it finished reading this band's rows
 * (count >= value * per-launch target). A rank
 * about to overwrite its band's input rows after step e enqueues
 * sc_band_signal_wait(above, below, 1, e, err, stream) first. */
int sc_band_signal_wait(const uint64_t *sig_above, const uint64_t *sig_below, int word, uint64_t value,
                        uint32_t *sig_err, void *stream);

/* NCCL transport of the row-band step (one process per GPU). The library loads
 * libnccl.so.2 at run time and keeps its own communicator:
 *   sc_nccl_unique_id   -> 128-byte ncclUniqueId on one rank (share it, e.g. by
 *                          torch.distributed broadcast)
 *   sc_nccl_comm_init   -> ncclCommInitRank on `device`
 * A band plan holds, for one band of `nplanes` planes (owned rows
 * [band_lo, band_hi) of a global_rows x cols image; src / dst hold exactly those
 * rows), ONE packed send and ONE receive buffer of nplanes x r x cols per
 * neighbour, a communication stream and, with use_graph, the whole step captured
 * in a CUDA graph (off by default in the Python layer: measured, the graph launch
 * with NCCL nodes costs the host more than the eager step's ~25 us). A step: pack the r boundary rows of every plane (one 2-D copy per
 * side) and exchange them (ncclSend/ncclRecv in one group) on the communication
 * stream while the interior rows [lo+r, hi-r) compute on the caller's stream;
 * then ONE launch produces both boundary strips, reading the halo rows straight
 * from the receive buffers. rank_above / rank_below: the neighbours' ranks (-1 at
 * the image edges; a rank may name itself, which the one-GPU tests use). */
int sc_nccl_unique_id(void *id_out /* 128 bytes */);
int sc_nccl_comm_init(const void *id /* 128 bytes */, int nranks, int rank, int device, void **comm_out);
int sc_nccl_comm_destroy(void *comm);
int sc_band_plan_create(void *comm, const float *src, float *dst, int nplanes, int global_rows, int cols,
                        int64_t src_plane_stride, int64_t dst_plane_stride, int64_t src_row_stride,
                        int64_t dst_row_stride, int band_lo, int band_hi, int rank_above, int rank_below,
                        const float *taps, int width, int flags, int use_graph, void **plan_out);
int sc_band_plan_step(void *plan, void *stream);
/* 1 if the plan's steps replay a captured CUDA graph, 0 if they are issued eagerly */
int sc_band_plan_graphed(void *plan);
int sc_band_plan_destroy(void *plan);

/* CUDA IPC for the band buffers: export a device buffer (64-byte handle of its
 * allocation + the buffer's byte offset in it), map another process's buffer for
 * use by `device` (peer access enabled on demand), and unmap it. */
int sc_ipc_export(const void *dev_ptr, void *handle_out /* 64 bytes */, int64_t *offset_out);
int sc_ipc_open(const void *handle /* 64 bytes */, int64_t offset, int device, void **ptr_out);
int sc_ipc_close(void *ptr, int64_t offset);

/* horizontal_rows_vec over rows [row_lo,row_hi) (S/conv.py:215-240; public
 * horizontal_pass uses [r, R-r), S/conv.py:362-375). SC_ZERO_FILL also zeroes
 * every other dst element (the two-pass scratch convention). */
int sc_hpass_f32(const float *src, float *dst, int nplanes, int rows, int cols,
                 int64_t src_plane_stride, int64_t dst_plane_stride,
                 int64_t src_row_stride, int64_t dst_row_stride,
                 int row_lo, int row_hi, const float *taps, int width, int flags, void *stream);

/* vertical_rows_vec over rows [row_lo,row_hi) within [r, R-r) (S/conv.py:269-293). */
int sc_vpass_f32(const float *src, float *dst, int nplanes, int rows, int cols,
                 int64_t src_plane_stride, int64_t dst_plane_stride,
                 int64_t src_row_stride, int64_t dst_row_stride,
                 int row_lo, int row_hi, const float *taps, int width, int flags, void *stream);

/* The reference two-pass with its exact buffer semantics: scratch := H0 (zero
 * outside the row-pass region), image[valid] := V(H0), image ring untouched.
 * conv_two_pass(plane, kernel, scratch, extended), S/conv.py:392-421.
 * 16-B aligned rows: ONE pass (image read once, both buffers written once; a
 * snapshot of the band/strip boundary samples is taken first, in a pooled
 * stream-ordered allocation). Otherwise, or with SC_SPLIT_PASSES=1: the row pass
 * with zero fill, then the column pass. */
int sc_two_pass_split_f32(float *image, float *scratch, int nplanes, int rows, int cols,
                          int64_t image_plane_stride, int64_t scratch_plane_stride,
                          int64_t image_row_stride, int64_t scratch_row_stride,
                          const float *taps, int width, int flags, void *stream);

/* The two-pass in place on device planes with NO observable scratch -- what
 * convolve_image(image, kernel, TWO_PASS, plan) does when the caller passes no
 * workspace (the reference then zeroes a fresh one nobody sees,
 * S/executors.py:303-304): image[valid] := V(H0), image ring untouched.
 * 16-B aligned rows: one pass over the image (2 traversals + the halo snapshot);
 * otherwise the row pass into a stream-ordered temporary + the column pass. */
int sc_two_pass_inplace_f32(float *image, int nplanes, int rows, int cols, int64_t plane_stride,
                            int64_t row_stride, const float *taps, int width, int flags, void *stream);

/* Single pass with the dense width x width matrix (row-major, pass the reference's
 * outer_product(k).matrix, S/kernels.py:66-72): dst[valid] := D, dst ring untouched
 * (single_pass_rows_vec S/conv.py:86-114 == unrolled5 :146-175). SC_COPY_BACK then
 * copies dst[valid] into src[valid] (S/executors.py:330-331). */
int sc_single_pass_f32(float *src, float *dst, int nplanes, int rows, int cols,
                       int64_t src_plane_stride, int64_t dst_plane_stride,
                       int64_t src_row_stride, int64_t dst_row_stride,
                       const float *dense, int width, int flags, void *stream);

/* copy_back (S/conv.py:424-440): dst[rows lo..hi, cols lo..hi] := src[...]. */
int sc_copy_region_f32(const float *src, float *dst, int nplanes, int rows, int cols,
                       int64_t src_plane_stride, int64_t dst_plane_stride,
                       int64_t src_row_stride, int64_t dst_row_stride,
                       int row_lo, int row_hi, int col_lo, int col_hi, void *stream);

/* Deterministic inputs: splitmix64 draw (offset+i) of `seed` (S/image.py:131-141)
 * mapped by kind: 0 -> [0,256) as make_synthetic (S/image.py:158-160),
 * 1 -> U[0,1), 2 -> U[0,255). */
int sc_fill_synthetic_f32(float *dst, int64_t count, uint64_t seed, uint64_t offset, int kind,
                          void *stream);

/* The PPM payload either side of the path (S/ppm.py): interleaved u8 HWC rows
 * (3 bytes per pixel, R,G,B = planes 0,1,2; row strides in BYTES).
 * sc_two_pass_u8hwc: read_ppm -> two-pass -> write_ppm fused, i.e. the bytes the
 * reference writes after convolve_image(TWO_PASS) on read_ppm(src)
 * (S/ppm.py:72-73, S/executors.py:308-326, S/ppm.py:87-89: rint half-even,
 * clip 0..255). Taps of width 1..9; any cols, row strides and byte offsets
 * (16-B aligned src rows with cols % 16 == 0 and a 4-B aligned dst run the
 * aligned build, anything else the general build: same bytes). */
int sc_two_pass_u8hwc(const uint8_t *src, uint8_t *dst, int rows, int cols, int64_t src_row_stride,
                      int64_t dst_row_stride, const float *taps, int width, int flags, void *stream);
/* u8 HWC -> 3 float32 planes (read_ppm_bytes, S/ppm.py:72-73). */
int sc_hwc_u8_to_planes_f32(const uint8_t *src, float *dst, int rows, int cols, int64_t src_row_stride,
                            int64_t dst_plane_stride, int64_t dst_row_stride, void *stream);
/* 3 float32 planes -> u8 HWC with clip(rint(x), 0, 255) (write_ppm_bytes, S/ppm.py:87-89). */
int sc_planes_f32_to_hwc_u8(const float *src, uint8_t *dst, int rows, int cols, int64_t src_plane_stride,
                            int64_t src_row_stride, int64_t dst_row_stride, void *stream);

/* End-to-end two-pass on HOST planes (the reference's Image: one pointer per
 * C-contiguous plane): streams row chunks H2D -> fused kernel -> D2H on three
 * CUDA streams with triple buffering, on `device`. In-place
 * (dst_planes == src_planes) is allowed, as in conv_two_pass. Pinned or
 * registered planes are copied by DMA directly; pageable planes go through a
 * pinned staging ring filled and drained by a pool of host threads (bound by
 * host memory bandwidth). Blocks until done. */
int sc_two_pass_host_f32(const float *const *src_planes, float *const *dst_planes, int nplanes,
                         int rows, int cols, const float *taps, int width, int flags, int device);

/* Page-lock (cudaHostRegister, portable) / release a caller's host range, so the
 * host entry points above DMA straight from / into it instead of staging it
 * through their pinned ring. The Python layer caches this per numpy buffer for
 * the buffer's lifetime (device.HostRegistry). */
int sc_host_register(void *ptr, int64_t bytes);
int sc_host_unregister(void *ptr);

/* The reference's exact end state of BOTH host buffers of
 * convolve_image(image, kernel, TWO_PASS, plan, workspace=workspace)
 * (S/executors.py:303-326): workspace := H0 (zeroed, then the row pass on rows
 * [r, R-r) or every row with SC_EXTENDED, cols [r, C-r)), image[valid] := V(H0)
 * in place, image ring untouched. Streams like sc_two_pass_host_f32 (each chunk
 * also writes its H0 rows back). Replaces the two per-plane phases the
 * reference's executor runs (horizontal then vertical rows, S/executors.py:318-323). */
int sc_two_pass_host_split_f32(float *const *image_planes, float *const *scratch_planes, int nplanes, int rows,
                               int cols, const float *taps, int width, int flags, int device);

/* Single pass over HOST planes: convolve_image's single-pass variants on numpy
 * planes (S/executors.py:327-356; bodies S/conv.py:86-114, :146-175).
 * workspace[valid] := the dense fold of the image (dense = width x width,
 * row-major: the reference's outer_product(kernel).matrix); with SC_COPY_BACK the
 * same samples also go back into image[valid] (S/conv.py:424-449), in place.
 * Everything else in both buffers keeps its values. The workspace must not
 * overlap the image. Streams like sc_two_pass_host_f32. */
int sc_single_pass_host_f32(float *const *image_planes, float *const *workspace_planes, int nplanes, int rows,
                            int cols, const float *dense, int width, int flags, int device);

/* sc_single_pass_host_f32 over several GPUs from one process: row bands by the
 * reference's balanced split (S/executors.py:121-139), one host thread and one
 * PCIe link per device, the rows around band boundaries copied aside first. */
int sc_single_pass_host_multi_f32(float *const *image_planes, float *const *workspace_planes, int nplanes,
                                  int rows, int cols, const float *dense, int width, int flags,
                                  const int *devices, int ndev);

/* horizontal_pass / vertical_pass on HOST planes (S/conv.py:362-389): dst[valid] :=
 * the row pass (vertical = 0) or the column pass (vertical != 0) of src over rows
 * [r, R-r) and columns [r, C-r); dst elsewhere keeps its values; dst must not
 * overlap src. Streams like sc_two_pass_host_f32. */
int sc_pass_host_f32(const float *const *src_planes, float *const *dst_planes, int nplanes, int rows, int cols,
                     const float *taps, int width, int vertical, int device);

/* Rows [out_lo, out_hi) only (one rank's row band of a host-resident image,
 * global-row rules): reads host rows [out_lo-r, out_hi+r) clipped to the image,
 * writes host rows [out_lo, out_hi); plane pointers address row 0 and no other
 * row is touched. Same streaming as sc_two_pass_host_f32 (which is the band
 * [0, rows)). */
int sc_two_pass_host_band_f32(const float *const *src_planes, float *const *dst_planes, int nplanes, int rows,
                              int cols, int out_lo, int out_hi, const float *taps, int width, int flags,
                              int device);

/* sc_two_pass_host_f32 over SEVERAL GPUs from one process (the reference's plans
 * are single-process): ndev row bands by the reference's balanced split
 * (partition_block, S/executors.py:121-139), each streamed through its own GPU
 * and PCIe link by its own host thread, concurrently. The 2r rows around every
 * band boundary are copied aside first, so in-place use stays exact. Same bits
 * as one device. A device may be listed more than once (its bands then run one
 * after the other). Blocks until done. */
int sc_two_pass_host_multi_f32(const float *const *src_planes, float *const *dst_planes, int nplanes, int rows,
                               int cols, const float *taps, int width, int flags, const int *devices, int ndev);

/* sc_two_pass_host_split_f32 over several GPUs from one process: the same row
 * bands as sc_two_pass_host_multi_f32, each writing its image rows (ring
 * untouched) and its workspace rows (H0); the reference's end state of both
 * buffers, same bits as one device. */
int sc_two_pass_host_multi_split_f32(float *const *image_planes, float *const *scratch_planes, int nplanes, int rows,
                                     int cols, const float *taps, int width, int flags, const int *devices, int ndev);

#ifdef __cplusplus
}
#endif

#endif /* SEPCONV_B200_H */
