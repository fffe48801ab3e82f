// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Flat C entry points over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libsdct_ref.so).
// Used only by tests/, bench.py's cpu_baseline / --impl reference legs and
// tests/golden/make_golden.py. The product path never links or loads this.
//
// Each entry builds the reference plan once (Plan2d / Plan3d, as the reference
// does per call in proj/src/dct2d.cpp:389-393) and then runs the transform
// `reps` times so a caller can time the prebuilt-plan path; the output of the
// last repetition is written to `out`.

#include <chrono>
#include <cstddef>
#include <cstring>
#include <exception>
#include <string>

#include "sdct/dct2d.hpp"
#include "sdct/errors.hpp"
#include "sdct/force.hpp"
#include "sdct/io.hpp"
#include "sdct/exec.hpp"
#include "sdct/transforms_ext.hpp"

namespace {

thread_local std::string g_err;

enum RefKind {
  REF_DCT2 = 0,
  REF_IDCT2 = 1,
  REF_IDCT_IDXST = 2,
  REF_IDXST_IDCT = 3,
  REF_DCT3 = 4,
  REF_IDCT3 = 5,
  REF_DCT2_ROWCOL = 6,
  REF_IDCT_IDXST_ROWCOL = 7,
  REF_IDXST_IDCT_ROWCOL = 8,
};

}  // namespace

extern "C" {

const char* sdct_ref_last_error() { return g_err.c_str(); }

// Returns 0 on success, 1 on shape errors, 2 on anything else.
int sdct_ref_run(int kind, int rank, const std::size_t* dims, const double* in, double* out,
                 unsigned threads, int reps) {
  try {
    sdct::ExecConfig cfg;
    cfg.parallelism_degree = threads;
    sdct::Shape shape(dims, dims + rank);
    sdct::RealTensor x(shape, std::vector<double>(in, in + sdct::numel(shape)));
    sdct::RealTensor y;
    if (kind == REF_DCT3 || kind == REF_IDCT3) {
      if (rank != 3) throw sdct::ShapeError("3D kinds need rank 3");
      sdct::Plan3d plan(dims[0], dims[1], dims[2]);
      for (int r = 0; r < reps; ++r)
        y = kind == REF_DCT3 ? sdct::dct_3d(x, plan, cfg) : sdct::idct_3d(x, plan, cfg);
    } else {
      if (rank != 2) throw sdct::ShapeError("2D kinds need rank 2");
      sdct::Plan2d plan(dims[0], dims[1]);
      for (int r = 0; r < reps; ++r) {
        switch (kind) {
          case REF_DCT2: y = sdct::dct_2d(x, plan, cfg); break;
          case REF_IDCT2: y = sdct::idct_2d(x, plan, cfg); break;
          case REF_IDCT_IDXST: y = sdct::idct_idxst_2d(x, plan, cfg); break;
          case REF_IDXST_IDCT: y = sdct::idxst_idct_2d(x, plan, cfg); break;
          case REF_DCT2_ROWCOL: y = sdct::dct_2d_rowcol(x, plan, cfg); break;
          case REF_IDCT_IDXST_ROWCOL: y = sdct::idct_idxst_2d_rowcol(x, plan, cfg); break;
          case REF_IDXST_IDCT_ROWCOL: y = sdct::idxst_idct_2d_rowcol(x, plan, cfg); break;
          default: throw sdct::ShapeError("unknown kind");
        }
      }
    }
    std::memcpy(out, y.data(), y.size() * sizeof(double));
    return 0;
  } catch (const sdct::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"

extern "C" {

// sdct::force_demo_fields (proj/src/force.cpp:11-37) on an n1 x n2 density.
int sdct_ref_force(std::size_t n1, std::size_t n2, const double* in, double* xi1, double* xi2, unsigned threads,
                   int reps) {
  try {
    sdct::ExecConfig cfg;
    cfg.parallelism_degree = threads;
    sdct::RealTensor x(sdct::Shape{n1, n2}, std::vector<double>(in, in + n1 * n2));
    sdct::ForceFields f;
    for (int r = 0; r < reps; ++r) f = sdct::force_demo_fields(x, cfg);
    std::memcpy(xi1, f.xi1.data(), n1 * n2 * sizeof(double));
    std::memcpy(xi2, f.xi2.data(), n1 * n2 * sizeof(double));
    return 0;
  } catch (const sdct::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"

extern "C" {

// sdct::write_dctb (proj/src/io.cpp:96-107) of a rank-`rank` tensor.
int sdct_ref_write_dctb(const char* path, int rank, const std::size_t* dims, const double* data) {
  try {
    sdct::Shape shape(dims, dims + rank);
    sdct::RealTensor x(shape, std::vector<double>(data, data + (rank ? sdct::numel(shape) : 0)));
    sdct::write_dctb(path, x);
    return 0;
  } catch (const sdct::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const sdct::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// sdct::read_dctb (proj/src/io.cpp:60-94): 0 and rank/dims (+ payload when
// cap >= numel) on success, 3 on FormatError.
int sdct_ref_read_dctb(const char* path, int* rank, std::size_t* dims, double* out, std::size_t cap) {
  try {
    const sdct::RealTensor x = sdct::read_dctb(path);
    *rank = static_cast<int>(x.rank());
    for (std::size_t d = 0; d < x.rank(); ++d) dims[d] = x.dim(d);
    if (out && cap >= x.size()) std::memcpy(out, x.data(), x.size() * sizeof(double));
    return 0;
  } catch (const sdct::FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const sdct::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"

extern "C" {

// Timed variants for bench.py's CPU arm: the plan is built once outside the
// clock (as a prebuilt-plan caller would hold it), the input tensor is built
// once, and only the `reps` transform calls are timed (steady_clock);
// *seconds = their total. The output of the last call lands in `out`.
int sdct_ref_run_timed(int kind, int rank, const std::size_t* dims, const double* in, double* out,
                       unsigned threads, int reps, double* seconds) {
  try {
    sdct::ExecConfig cfg;
    cfg.parallelism_degree = threads;
    sdct::Shape shape(dims, dims + rank);
    sdct::RealTensor x(shape, std::vector<double>(in, in + sdct::numel(shape)));
    sdct::RealTensor y;
    std::chrono::steady_clock::time_point t0;
    if (kind == REF_DCT3 || kind == REF_IDCT3) {
      if (rank != 3) throw sdct::ShapeError("3D kinds need rank 3");
      sdct::Plan3d plan(dims[0], dims[1], dims[2]);
      t0 = std::chrono::steady_clock::now();
      for (int r = 0; r < reps; ++r)
        y = kind == REF_DCT3 ? sdct::dct_3d(x, plan, cfg) : sdct::idct_3d(x, plan, cfg);
    } else {
      if (rank != 2) throw sdct::ShapeError("2D kinds need rank 2");
      sdct::Plan2d plan(dims[0], dims[1]);
      t0 = std::chrono::steady_clock::now();
      for (int r = 0; r < reps; ++r) {
        switch (kind) {
          case REF_DCT2: y = sdct::dct_2d(x, plan, cfg); break;
          case REF_IDCT2: y = sdct::idct_2d(x, plan, cfg); break;
          case REF_IDCT_IDXST: y = sdct::idct_idxst_2d(x, plan, cfg); break;
          case REF_IDXST_IDCT: y = sdct::idxst_idct_2d(x, plan, cfg); break;
          case REF_DCT2_ROWCOL: y = sdct::dct_2d_rowcol(x, plan, cfg); break;
          case REF_IDCT_IDXST_ROWCOL: y = sdct::idct_idxst_2d_rowcol(x, plan, cfg); break;
          case REF_IDXST_IDCT_ROWCOL: y = sdct::idxst_idct_2d_rowcol(x, plan, cfg); break;
          default: throw sdct::ShapeError("unknown kind");
        }
      }
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(out, y.data(), y.size() * sizeof(double));
    return 0;
  } catch (const sdct::ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// sdct::force_demo_fields timed the same way (input built once, calls timed).
int sdct_ref_force_timed(std::size_t n1, std::size_t n2, const double* in, double* xi1, double* xi2,
                         unsigned threads, int reps, double* seconds) {
  try {
    sdct::ExecConfig cfg;
    cfg.parallelism_degree = threads;
    sdct::RealTensor x(sdct::Shape{n1, n2}, std::vector<double>(in, in + n1 * n2));
    sdct::ForceFields f;
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) f = sdct::force_demo_fields(x, cfg);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(xi1, f.xi1.data(), n1 * n2 * sizeof(double));
    std::memcpy(xi2, f.xi2.data(), n1 * n2 * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
