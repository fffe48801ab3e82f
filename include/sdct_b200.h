/*
 * sdct_b200.h — C ABI of the B200-native multi-dimensional DCT library.
 *
 * This is the drop-in boundary for the reference's hot path (arXiv 2110.01172
 * three-stage DCT; reference C++ API in /root/reference/proj/include/sdct and
 * its pybind11 module proj/bindings/module.cpp). Plain pointers, sizes and
 * integer status codes only: no C++ or torch types cross this boundary.
 *
 * Conventions (identical to the reference, proj/include/sdct/dct2d.hpp:1-19,
 * transforms_ext.hpp:1-15): unnormalised cosine sums, row-major, extents
 * outermost first.
 *   DCT_2D        y = sum x cos cos              (== scipy dctn type 2 / 4)
 *   IDCT_2D       idct_2d(dct_2d(x)) == N1 N2 / 4 x
 *   IDCT_IDXST_2D IDCT along axis 0, IDXST along axis 1
 *   IDXST_IDCT_2D IDXST along axis 0, IDCT along axis 1
 *   DCT_3D        == dctn / 8;  IDCT_3D: idct_3d(dct_3d(x)) == N1 N2 N3 / 8 x
 *
 * A plan describes one shape, one dtype and a leading batch count; every
 * transform of the plan runs out of place on `batch` contiguous items.
 * Device entry points are stream-ordered and asynchronous; host entry points
 * copy through the plan's staging buffers and synchronise.
 */
#ifndef SDCT_B200_H_
#define SDCT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ shim (include/sdct/errors.hpp) rethrows them as the
 * reference's exception types (proj/include/sdct/errors.hpp:11-33):
 * SHAPE -> ShapeError, PLAN -> PlanError (is-a ShapeError), BOUNDS ->
 * BoundsError; the pybind module maps ShapeError to ValueError exactly like
 * proj/bindings/module.cpp:64-65. */
enum {
  SDCT_OK = 0,
  SDCT_ERR_SHAPE = 1,    /* rank/extent invalid                           */
  SDCT_ERR_PLAN = 2,     /* input does not match the plan                 */
  SDCT_ERR_BOUNDS = 3,   /* index out of range (corrupt-twiddle hook)     */
  SDCT_ERR_CUDA = 4,     /* CUDA runtime failure (message has the detail) */
  SDCT_ERR_OOM = 5,      /* device allocation failed                      */
  SDCT_ERR_ARG = 6,      /* null pointer / unknown enum                   */
  SDCT_ERR_NODEVICE = 7  /* no usable CUDA device                         */
};

enum { SDCT_F32 = 0, SDCT_F64 = 1 };

/* Orientation of a 2D plan (proj/include/sdct/dct2d.hpp:26, 43-46). The GPU
 * pipeline computes the same transform for both; the value is recorded so
 * Plan2d::orientation() keeps the reference's meaning. -1 = automatic
 * (maybe_transpose_strategy, proj/src/dct2d.cpp:294-298). */
enum { SDCT_ORIENT_AUTO = -1, SDCT_ORIENT_DIRECT = 0, SDCT_ORIENT_TRANSPOSED = 1 };

/* Transform kinds; each replaces the named reference entry point. */
enum {
  SDCT_DCT_2D = 0,        /* sdct::dct_2d        proj/include/sdct/dct2d.hpp:105-107 */
  SDCT_IDCT_2D = 1,       /* sdct::idct_2d       proj/include/sdct/dct2d.hpp:115-117 */
  SDCT_IDCT_IDXST_2D = 2, /* sdct::idct_idxst_2d proj/include/sdct/transforms_ext.hpp:34-35 */
  SDCT_IDXST_IDCT_2D = 3, /* sdct::idxst_idct_2d proj/include/sdct/transforms_ext.hpp:36-37 */
  SDCT_DCT_3D = 4,        /* sdct::dct_3d        proj/include/sdct/transforms_ext.hpp:77-79 */
  SDCT_IDCT_3D = 5,       /* sdct::idct_3d       proj/include/sdct/transforms_ext.hpp:82-84 */
  SDCT_DCT_2D_ROWCOL = 6, /* sdct::dct_2d_rowcol proj/include/sdct/dct2d.hpp:111-112 */
  SDCT_DCT_1D = 7,        /* sdct::dct_1d        proj/include/sdct/dct1d.hpp:90-93  (rank-1 plans) */
  SDCT_IDCT_1D = 8,       /* sdct::idct_1d       proj/include/sdct/dct1d.hpp:97-99  (rank-1 plans) */
  SDCT_IDXST_1D = 9,      /* sdct::idxst_1d      proj/include/sdct/transforms_ext.hpp:29-31 */
  SDCT_IDCT_IDXST_2D_ROWCOL = 10, /* sdct::idct_idxst_2d_rowcol proj/include/sdct/transforms_ext.hpp:43-44 */
  SDCT_IDXST_IDCT_2D_ROWCOL = 11, /* sdct::idxst_idct_2d_rowcol proj/include/sdct/transforms_ext.hpp:45-46 */
  SDCT_DCT_AXIS0 = 12,    /* sdct::dct_1d (N-point, proj/src/dct1d.cpp) of every column of a rank-2 plan */
  SDCT_IDCT_AXIS0 = 13    /* sdct::idct_1d of every column of a rank-2 plan */
};
/* The two *_AXIS0 kinds are the axis-0 leg of the slab-decomposed 3D transform
 * (SURVEY.md §8e): one persistent column pass over an (n1 x n2) matrix, n1 a
 * power of two in [8, 4096], n2 a multiple of 32 bytes' worth of elements. */
/* The three *_ROWCOL kinds are the reference's 8-stage row-column baselines
 * (proj/src/dct2d.cpp:395-406, transforms_ext.cpp:287-311): per axis one
 * kernel (parity reorder / embedding, row FFTs and twiddle stage fused) and
 * one tiled transpose — 4 launches, 4 HBM round trips of the tensor. */

typedef struct sdct_plan_s* sdct_plan_t;

/* Library version (major*10000 + minor*100 + patch). */
int sdct_version(void);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* sdct_last_error(void);

/* Plan construction — replaces sdct::Plan2d::Plan2d (proj/src/dct2d.cpp:300-306),
 * sdct::Plan3d::Plan3d (proj/src/transforms_ext.cpp:313-320) and
 * sdct::Plan1d (proj/include/sdct/dct1d.hpp:35-52). rank is 1, 2 or 3; dims
 * holds rank positive extents; batch >= 1 items of that shape are processed
 * per call. Builds the per-shape device twiddle tables and launch geometry on
 * `device` (-1 = current device). Extents <= 0 give SDCT_ERR_SHAPE (the
 * reference throws ShapeError, dct2d.cpp:12-15). */
int sdct_plan_create(sdct_plan_t* plan, int rank, const int64_t* dims, int64_t batch, int dtype,
                     int orientation, int device);
int sdct_plan_destroy(sdct_plan_t plan);

/* Plan facts: orientation actually used (Plan2d::orientation()), whether the
 * power-of-two fast kernels serve this shape (1) or the generic path (0),
 * and the device workspace bytes sdct_exec needs when the caller supplies one. */
int sdct_plan_orientation(sdct_plan_t plan, int* orientation);
int sdct_plan_is_fast(sdct_plan_t plan, int* fast);
int sdct_plan_workspace_size(sdct_plan_t plan, size_t* bytes);
/* Device memory the plan currently owns (tables, and whatever it allocated on
 * first use: its own workspace, host staging, pipeline lanes, scratch). Plan
 * caches (C++ make_plan, Python plan_for) bound their footprint with it. */
int sdct_plan_device_bytes(sdct_plan_t plan, size_t* bytes);

/* Test-only fault injection: negates axis-1 twiddle b[index] (2D) exactly like
 * sdct::Plan2d::corrupt_twiddle_for_testing (proj/src/dct2d.cpp:312-317);
 * index >= N2 gives SDCT_ERR_BOUNDS. */
int sdct_plan_corrupt_twiddle(sdct_plan_t plan, int64_t index);

/* Run one transform on device memory, stream-ordered. d_in/d_out hold
 * batch*numel elements of the plan dtype (distinct buffers). d_workspace may
 * be NULL (the plan's own workspace is used; concurrent calls on one plan then
 * need distinct streams serialised by the caller) or a buffer of
 * sdct_plan_workspace_size bytes. stream is a cudaStream_t (NULL = default). */
int sdct_exec(sdct_plan_t plan, int kind, const void* d_in, void* d_out, void* d_workspace,
              void* stream);

/* Same transform on host memory: copies in (H2D), runs, copies out (D2H) and
 * synchronises `stream`. This is what the C++ value API (RealTensor in,
 * RealTensor out, proj/include/sdct/tensor.hpp:34-78) calls. */
int sdct_exec_host(sdct_plan_t plan, int kind, const void* h_in, void* h_out, void* stream);

/* DREAMPlace-style spectral force fields — replaces sdct::force_demo_fields
 * (proj/src/force.cpp:11-37, proj/include/sdct/force.hpp:23): a = dct_2d(density),
 * a1 = a w1/(w1^2+w2^2), a2 = a w2/(w1^2+w2^2) (w_d = pi k_d / n_d, 0 at DC),
 * xi1 = idct_idxst_2d(a1), xi2 = idxst_idct_2d(a2). Device buffers of one
 * plan-sized batch; the weighting is fused into the inverse passes' loads (no
 * a1/a2 arrays). d_workspace as for sdct_exec (NULL = the plan's own).
 * Stream-ordered; the coefficients live in a plan-owned scratch buffer, so
 * concurrent calls on one plan must be ordered by the caller (one stream). */
int sdct_force_fields(sdct_plan_t plan, const void* d_density, void* d_xi1, void* d_xi2, void* d_workspace,
                      void* stream);
/* Bytes of the caller-provided coefficient scratch that sdct_force_fields_scratch
 * and sdct_compress_scratch take (0 for plans of rank != 2). */
int sdct_scratch_size(sdct_plan_t plan, size_t* bytes);
/* sdct_force_fields with the coefficient / intermediate scratch in d_scratch
 * (256-byte aligned, sdct_scratch_size bytes; NULL = the plan-owned buffer):
 * with a scratch per call, concurrent calls on one plan from different streams
 * are safe. */
int sdct_force_fields_scratch(sdct_plan_t plan, const void* d_density, void* d_xi1, void* d_xi2, void* d_workspace,
                              void* d_scratch, void* stream);
/* Same on host memory (H2D, the fused device pipeline, D2H, synchronised). */
int sdct_force_fields_host(sdct_plan_t plan, const void* h_density, void* h_xi1, void* h_xi2, void* stream);

/* Whole-image frequency-domain compression — the numeric core of
 * sdct::compress_image (proj/src/compress.cpp:24-54): b = dct_2d(image); every
 * coefficient with |b| < epsilon (raw, unnormalised magnitudes) is zeroed and
 * counted into *d_zeroed (a device counter the caller zeroes; may be NULL);
 * d_out = idct_2d(b) * 4/(N1 N2). The threshold and the normalisation ride on
 * the inverse row kernels' loads. Rounding to 8-bit samples and PSNR are the
 * image app's (out of scope). epsilon may be +inf; < 0 or NaN -> SDCT_ERR_ARG.
 * Shares the plan-owned coefficient scratch with sdct_force_fields (order
 * concurrent calls on one plan). */
int sdct_compress(sdct_plan_t plan, const void* d_in, void* d_out, double epsilon, unsigned long long* d_zeroed,
                  void* d_workspace, void* stream);
/* sdct_compress with a caller-provided scratch (as sdct_force_fields_scratch). */
int sdct_compress_scratch(sdct_plan_t plan, const void* d_in, void* d_out, double epsilon,
                          unsigned long long* d_zeroed, void* d_workspace, void* d_scratch, void* stream);

/* Host streaming: `count` independent items (each one plan-sized batch) go
 * host -> device -> kinds[0] -> ... -> kinds[nkinds-1] -> host. Item i's input
 * is at h_in + i*in_stride bytes and its result is written to
 * h_out + i*out_stride (stride 0 reuses one buffer). The items are software
 * pipelined over three internal streams with their own device buffers, so
 * item i+1's H2D, item i's kernels and item i-1's D2H overlap (PCIe is full
 * duplex). Stream-ordered on `stream` (fork/join through events): the call
 * returns once everything is queued; results are in h_out when `stream`
 * reaches that point. Host buffers must be pinned for the copies to overlap.
 * The batched-host counterpart of calling dct_2d (proj/src/dct2d.cpp:389-393)
 * once per image. */
int sdct_exec_host_pipelined(sdct_plan_t plan, const int* kinds, int nkinds, const void* h_in, int64_t in_stride,
                             void* h_out, int64_t out_stride, int64_t count, void* stream);

/* Batched transpose of device memory: `batch` items of rows x cols (dtype
 * SDCT_F32/F64) become cols x rows, out of place, stream-ordered. The axis
 * regrouping of the reference's rank-4 factorisation (transpose_2d inside
 * proj/src/transforms_ext.cpp:396-425) and the row-column kinds use it. */
int sdct_transpose(int dtype, int64_t rows, int64_t cols, int64_t batch, const void* d_in, void* d_out,
                   void* stream);

/* Stage-level real FFTs with the reference's HalfSpectrum layout — replace
 * sdct::rfft_nd / irfft_nd (proj/include/sdct/rfft.hpp:66-70, rfft.cpp:182-245):
 * unnormalised, kernel e^{-2 pi i nk/N}, one-sided (last/2 + 1 complex entries,
 * interleaved re/im doubles) along the last axis, full along the others.
 * The plan gives rank (1..3), extents and batch; fp64 plans only (the
 * reference is fp64). d_workspace: NULL (plan-owned scratch; serialise
 * concurrent calls on one plan) or sdct_rfft_workspace_size bytes. The
 * inverse treats the stored half as authoritative and keeps the real part. */
int sdct_rfft_workspace_size(sdct_plan_t plan, size_t* bytes);
int sdct_rfft_nd(sdct_plan_t plan, const void* d_x, void* d_half, void* d_workspace, void* stream);
int sdct_irfft_nd(sdct_plan_t plan, const void* d_half, void* d_x, void* d_workspace, void* stream);
/* Host-memory versions (copy in, run, copy out, synchronise). */
int sdct_rfft_nd_host(sdct_plan_t plan, const double* h_x, double* h_half);
int sdct_irfft_nd_host(sdct_plan_t plan, const double* h_half, double* h_x);
/* O(n^2) direct DFT of n complex values on the GPU (sdct::dft_naive,
 * proj/src/rfft.cpp:113-127, the backend's own reference); host buffers. */
int sdct_dft_naive_host(int64_t n, int inverse, const double* h_in, double* h_out);

/* Stage-level access for timing the individual kernels of a transform:
 * number of kernel launches of `kind`, and a launch of one of them with the
 * same argument meaning as sdct_exec (stage k reads/writes the buffers the
 * full pipeline would). */
int sdct_stage_count(sdct_plan_t plan, int kind, int* count);
int sdct_exec_stage(sdct_plan_t plan, int kind, int stage, const void* d_in, void* d_out,
                    void* d_workspace, void* stream);

/* Analytic sdct::StageCounters (proj/include/sdct/exec.hpp:29-50) for one
 * call of `kind`: full_tensor_stages, element_reads, element_writes,
 * real_mults, real_adds — the values the reference's Counted kernels tally
 * (proj/src/dct2d.cpp:48-238), computed from the plan's shape. */
int sdct_counters(sdct_plan_t plan, int kind, uint64_t out[5]);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* SDCT_B200_H_ */
