// pybind11 module `_sdct`: the reference's Python surface
// (proj/bindings/module.cpp:62-171, proj/python/sdct/__init__.py:8-26) over
// the C++ API, plus `Plan`, a device-memory plan for torch tensors / raw
// device pointers. numpy in -> float64 numpy out with copies, exactly like
// the reference; ShapeError / FormatError subclass ValueError
// (module.cpp:64-65). The GIL is released while the GPU works.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <stdexcept>
#include <string>

#include "sdct/dct1d.hpp"
#include "sdct/dct2d.hpp"
#include "sdct/force.hpp"
#include "sdct/device.hpp"
#include "sdct/errors.hpp"
#include "sdct/transforms_ext.hpp"
#include "sdct/plan_handle.hpp"
#include "sdct_b200.h"

namespace py = pybind11;

namespace {

using Array = py::array_t<double, py::array::c_style | py::array::forcecast>;

sdct::RealTensor to_tensor(const Array& a) {
  const py::buffer_info info = a.request();
  if (info.ndim < 1 || info.ndim > 4)
    throw sdct::ShapeError("expected a rank 1..4 array, got rank " + std::to_string(info.ndim));
  sdct::Shape dims;
  for (py::ssize_t d : info.shape) {
    if (d <= 0) throw sdct::ShapeError("tensor extents must be positive");
    dims.push_back(static_cast<std::size_t>(d));
  }
  const double* p = static_cast<const double*>(info.ptr);
  return sdct::RealTensor(dims, std::vector<double>(p, p + info.size));
}

Array to_array(const sdct::RealTensor& t) {
  std::vector<py::ssize_t> shape(t.dims().begin(), t.dims().end());
  Array out(shape);
  std::copy(t.data(), t.data() + t.size(), static_cast<double*>(out.request().ptr));
  return out;
}

template <typename F>
Array run(const Array& x, F&& f) {
  sdct::RealTensor t = to_tensor(x);
  sdct::RealTensor y;
  {
    py::gil_scoped_release nogil;
    y = f(t);
  }
  return to_array(y);
}

// Fused 2D/3D transforms straight between the numpy buffers: the input
// array (already float64 C-contiguous after forcecast) goes to the device
// plan's host entry point and the result lands in the freshly allocated
// output array, with no RealTensor copies in between. Same plan (cache key
// and orientation) the C++ API's Plan2d / Plan3d would use; any other rank
// takes the C++ API path, which raises the reference's ShapeError.
template <typename F>
Array run_fused(const Array& x, int rank, int kind, F&& fallback) {
  const py::buffer_info info = x.request();
  bool ok = info.ndim == rank;
  for (py::ssize_t d : info.shape) ok = ok && d > 0;
  if (!ok) return run(x, fallback);
  std::vector<std::int64_t> dims(info.shape.begin(), info.shape.end());
  const int orient = rank == 2 ? (sdct::maybe_transpose_strategy(static_cast<std::size_t>(dims[0]),
                                                                 static_cast<std::size_t>(dims[1])) ==
                                          sdct::Orientation::Direct
                                      ? SDCT_ORIENT_DIRECT
                                      : SDCT_ORIENT_TRANSPOSED)
                               : SDCT_ORIENT_DIRECT;
  Array out(std::vector<py::ssize_t>(info.shape.begin(), info.shape.end()));
  double* po = static_cast<double*>(out.request().ptr);
  const double* pi = static_cast<const double*>(info.ptr);
  {
    py::gil_scoped_release nogil;
    sdct::detail::PlanPtr plan = sdct::detail::make_plan(dims, 1, SDCT_F64, orient);
    sdct::detail::check(sdct_exec_host(plan.get(), kind, pi, po, nullptr));
  }
  return out;
}

sdct::Dct1dVariant variant_from_name(const std::string& name) {
  if (name == "4n") return sdct::Dct1dVariant::FourN;
  if (name == "2n-mirrored") return sdct::Dct1dVariant::MirroredTwoN;
  if (name == "2n-padded") return sdct::Dct1dVariant::PaddedTwoN;
  if (name == "n") return sdct::Dct1dVariant::NPoint;
  throw std::invalid_argument("unknown variant '" + name +
                              "' (expected '4n', '2n-mirrored', '2n-padded' or 'n')");
}

}  // namespace

PYBIND11_MODULE(_sdct, m) {
  m.doc() = "B200-native multi-dimensional DCT/IDCT and IDXST/IDCT composites (sm_100a)";

  py::register_exception<sdct::ShapeError>(m, "ShapeError", PyExc_ValueError);
  py::register_exception<sdct::FormatError>(m, "FormatError", PyExc_ValueError);
  py::register_exception<sdct::DeviceError>(m, "DeviceError", PyExc_RuntimeError);

  m.def("dct_1d",
        [](const Array& x, const std::string& variant, unsigned) {
          const auto v = variant_from_name(variant);
          return run(x, [&](const sdct::RealTensor& t) { return sdct::dct_1d(t, v); });
        },
        py::arg("x"), py::arg("variant") = "n", py::arg("threads") = 0,
        "Forward 1D DCT, y(k) = sum_n x(n) cos(pi/N (n+1/2) k)");
  m.def("idct_1d",
        [](const Array& x, unsigned) { return run(x, [](const sdct::RealTensor& t) { return sdct::idct_1d(t); }); },
        py::arg("x"), py::arg("threads") = 0, "Inverse 1D DCT (idct_1d(dct_1d(x)) == N/2 * x)");
  m.def("idxst_1d",
        [](const Array& x, unsigned) { return run(x, [](const sdct::RealTensor& t) { return sdct::idxst_1d(t); }); },
        py::arg("x"), py::arg("threads") = 0, "y(k) = sum_{n>=1} x(n) sin(pi/N n (k+1/2))");

  m.def("dct_2d",
        [](const Array& x, unsigned) {
          return run_fused(x, 2, SDCT_DCT_2D, [](const sdct::RealTensor& t) { return sdct::dct_2d(t); });
        },
        py::arg("x"), py::arg("threads") = 0, "Fused forward 2D DCT on the B200");
  m.def("dct_2d_rowcol",
        [](const Array& x, unsigned) {
          return run(x, [](const sdct::RealTensor& t) {
            if (t.rank() != 2) throw sdct::ShapeError("dct_2d_rowcol expects a rank-2 array");
            return sdct::dct_2d_rowcol(t, sdct::Plan2d(t.dim(0), t.dim(1)));
          });
        },
        py::arg("x"), py::arg("threads") = 0, "Row-column 2D DCT (same output as dct_2d)");
  m.def("idct_idxst_2d_rowcol",
        [](const Array& x, unsigned) {
          return run(x, [](const sdct::RealTensor& t) {
            if (t.rank() != 2) throw sdct::ShapeError("idct_idxst_2d_rowcol expects a rank-2 array");
            return sdct::idct_idxst_2d_rowcol(t, sdct::Plan2d(t.dim(0), t.dim(1)));
          });
        },
        py::arg("x"), py::arg("threads") = 0, "Row-column IDCT/IDXST composite (same output as idct_idxst_2d)");
  m.def("idxst_idct_2d_rowcol",
        [](const Array& x, unsigned) {
          return run(x, [](const sdct::RealTensor& t) {
            if (t.rank() != 2) throw sdct::ShapeError("idxst_idct_2d_rowcol expects a rank-2 array");
            return sdct::idxst_idct_2d_rowcol(t, sdct::Plan2d(t.dim(0), t.dim(1)));
          });
        },
        py::arg("x"), py::arg("threads") = 0, "Row-column IDXST/IDCT composite (same output as idxst_idct_2d)");
  m.def("idct_2d",
        [](const Array& x, unsigned) {
          return run_fused(x, 2, SDCT_IDCT_2D, [](const sdct::RealTensor& t) { return sdct::idct_2d(t); });
        },
        py::arg("x"), py::arg("threads") = 0, "Fused inverse 2D DCT (idct_2d(dct_2d(x)) == N1*N2/4 * x)");
  m.def("idct_idxst_2d",
        [](const Array& x, unsigned) {
          return run_fused(x, 2, SDCT_IDCT_IDXST_2D, [](const sdct::RealTensor& t) {
            if (t.rank() != 2) throw sdct::ShapeError("idct_idxst_2d expects a rank-2 array");
            return sdct::idct_idxst_2d(t, sdct::Plan2d(t.dim(0), t.dim(1)));
          });
        },
        py::arg("x"), py::arg("threads") = 0, "IDCT along axis 0, IDXST along axis 1 (fused)");
  m.def("idxst_idct_2d",
        [](const Array& x, unsigned) {
          return run_fused(x, 2, SDCT_IDXST_IDCT_2D, [](const sdct::RealTensor& t) {
            if (t.rank() != 2) throw sdct::ShapeError("idxst_idct_2d expects a rank-2 array");
            return sdct::idxst_idct_2d(t, sdct::Plan2d(t.dim(0), t.dim(1)));
          });
        },
        py::arg("x"), py::arg("threads") = 0, "IDXST along axis 0, IDCT along axis 1 (fused)");
  m.def("dct_3d",
        [](const Array& x, unsigned) {
          return run_fused(x, 3, SDCT_DCT_3D, [](const sdct::RealTensor& t) { return sdct::dct_3d(t); });
        },
        py::arg("x"), py::arg("threads") = 0, "Fused forward 3D DCT on the B200");
  m.def("idct_3d",
        [](const Array& x, unsigned) {
          return run_fused(x, 3, SDCT_IDCT_3D, [](const sdct::RealTensor& t) { return sdct::idct_3d(t); });
        },
        py::arg("x"), py::arg("threads") = 0, "Fused inverse 3D DCT (idct_3d(dct_3d(x)) == N1*N2*N3/8 * x)");

  m.def("force_demo_fields",
        [](const Array& density, unsigned) {
          sdct::ForceFields f;
          {
            const sdct::RealTensor t = to_tensor(density);
            py::gil_scoped_release nogil;
            f = sdct::force_demo_fields(t);
          }
          return py::make_tuple(to_array(f.xi1), to_array(f.xi2));
        },
        py::arg("density"), py::arg("threads") = 0,
        "Inverse-Laplacian-weighted gradient fields (xi1, xi2) of a rank-2 density grid");

  m.def("amdahl_speedup",
        [](double p, double s) {
          if (!(p >= 0.0 && p <= 1.0)) throw std::invalid_argument("parallel fraction p must lie in [0, 1]");
          if (!(s > 0.0)) throw std::invalid_argument("speedup s must be positive");
          return 1.0 / ((1.0 - p) + p / s);
        },
        py::arg("p"), py::arg("s"), "1 / ((1 - p) + p / s)");

  // ---- device-memory plans --------------------------------------------------
  m.def("plan_cache_entries", &sdct::detail::plan_cache_entries,
        "Device plans held by the C++ plan cache (shared by the numpy entry points)");

  py::class_<sdct::DevicePlan>(m, "Plan")
      .def(py::init([](const std::vector<std::int64_t>& dims, std::int64_t batch, const std::string& dtype) {
             sdct::Dtype dt;
             if (dtype == "float32") dt = sdct::Dtype::F32;
             else if (dtype == "float64") dt = sdct::Dtype::F64;
             else throw std::invalid_argument("dtype must be 'float32' or 'float64'");
             return sdct::DevicePlan(dims, batch, dt);
           }),
           py::arg("dims"), py::arg("batch") = 1, py::arg("dtype") = "float64")
      .def("run",
           [](const sdct::DevicePlan& p, int kind, std::uintptr_t in, std::uintptr_t out, std::uintptr_t stream,
              std::uintptr_t ws) {
             py::gil_scoped_release nogil;
             p.run(kind, reinterpret_cast<const void*>(in), reinterpret_cast<void*>(out),
                   reinterpret_cast<void*>(stream), reinterpret_cast<void*>(ws));
           },
           py::arg("kind"), py::arg("d_in"), py::arg("d_out"), py::arg("stream") = 0, py::arg("workspace") = 0)
      .def("run_stage",
           [](const sdct::DevicePlan& p, int kind, int stage, std::uintptr_t in, std::uintptr_t out,
              std::uintptr_t stream, std::uintptr_t ws) {
             py::gil_scoped_release nogil;
             sdct::detail::check(sdct_exec_stage(p.handle(), kind, stage, reinterpret_cast<const void*>(in),
                                                 reinterpret_cast<void*>(out), reinterpret_cast<void*>(ws),
                                                 reinterpret_cast<void*>(stream)));
           },
           py::arg("kind"), py::arg("stage"), py::arg("d_in"), py::arg("d_out"), py::arg("stream") = 0,
           py::arg("workspace") = 0)
      .def("run_host_pipelined",
           [](const sdct::DevicePlan& p, const std::vector<int>& kinds, std::uintptr_t h_in, std::int64_t in_stride,
              std::uintptr_t h_out, std::int64_t out_stride, std::int64_t count, std::uintptr_t stream) {
             py::gil_scoped_release nogil;
             sdct::detail::check(sdct_exec_host_pipelined(
                 p.handle(), kinds.data(), static_cast<int>(kinds.size()), reinterpret_cast<const void*>(h_in),
                 in_stride, reinterpret_cast<void*>(h_out), out_stride, count, reinterpret_cast<void*>(stream)));
           },
           py::arg("kinds"), py::arg("h_in"), py::arg("in_stride"), py::arg("h_out"), py::arg("out_stride"),
           py::arg("count"), py::arg("stream") = 0)
      .def("force_fields",
           [](const sdct::DevicePlan& p, std::uintptr_t d_density, std::uintptr_t d_xi1, std::uintptr_t d_xi2,
              std::uintptr_t stream, std::uintptr_t ws, std::uintptr_t scratch) {
             py::gil_scoped_release nogil;
             sdct::detail::check(sdct_force_fields_scratch(
                 p.handle(), reinterpret_cast<const void*>(d_density), reinterpret_cast<void*>(d_xi1),
                 reinterpret_cast<void*>(d_xi2), reinterpret_cast<void*>(ws), reinterpret_cast<void*>(scratch),
                 reinterpret_cast<void*>(stream)));
           },
           py::arg("d_density"), py::arg("d_xi1"), py::arg("d_xi2"), py::arg("stream") = 0, py::arg("workspace") = 0,
           py::arg("scratch") = 0)
      .def("compress",
           [](const sdct::DevicePlan& p, std::uintptr_t d_in, std::uintptr_t d_out, double eps, std::uintptr_t d_zeroed,
              std::uintptr_t stream, std::uintptr_t ws, std::uintptr_t scratch) {
             py::gil_scoped_release nogil;
             sdct::detail::check(sdct_compress_scratch(p.handle(), reinterpret_cast<const void*>(d_in),
                                                       reinterpret_cast<void*>(d_out), eps,
                                                       reinterpret_cast<unsigned long long*>(d_zeroed),
                                                       reinterpret_cast<void*>(ws), reinterpret_cast<void*>(scratch),
                                                       reinterpret_cast<void*>(stream)));
           },
           py::arg("d_in"), py::arg("d_out"), py::arg("epsilon"), py::arg("d_zeroed") = 0, py::arg("stream") = 0,
           py::arg("workspace") = 0, py::arg("scratch") = 0)
      .def("stage_count",
           [](const sdct::DevicePlan& p, int kind) {
             int n = 0;
             sdct::detail::check(sdct_stage_count(p.handle(), kind, &n));
             return n;
           })
      .def_property_readonly("workspace_bytes", &sdct::DevicePlan::workspace_bytes)
      .def_property_readonly("device_bytes", &sdct::DevicePlan::device_bytes)
      .def_property_readonly("fast", &sdct::DevicePlan::fast)
      .def_property_readonly("scratch_bytes", [](const sdct::DevicePlan& p) {
        size_t b = 0;
        sdct::detail::check(sdct_scratch_size(p.handle(), &b));
        return b;
      });

  m.attr("DCT_2D") = py::int_(static_cast<int>(SDCT_DCT_2D));
  m.attr("IDCT_2D") = py::int_(static_cast<int>(SDCT_IDCT_2D));
  m.attr("IDCT_IDXST_2D") = py::int_(static_cast<int>(SDCT_IDCT_IDXST_2D));
  m.attr("IDXST_IDCT_2D") = py::int_(static_cast<int>(SDCT_IDXST_IDCT_2D));
  m.attr("DCT_3D") = py::int_(static_cast<int>(SDCT_DCT_3D));
  m.attr("IDCT_3D") = py::int_(static_cast<int>(SDCT_IDCT_3D));
  m.attr("DCT_2D_ROWCOL") = py::int_(static_cast<int>(SDCT_DCT_2D_ROWCOL));
  m.attr("IDCT_IDXST_2D_ROWCOL") = py::int_(static_cast<int>(SDCT_IDCT_IDXST_2D_ROWCOL));
  m.attr("IDXST_IDCT_2D_ROWCOL") = py::int_(static_cast<int>(SDCT_IDXST_IDCT_2D_ROWCOL));
  m.attr("DCT_AXIS0") = py::int_(static_cast<int>(SDCT_DCT_AXIS0));
  m.attr("IDCT_AXIS0") = py::int_(static_cast<int>(SDCT_IDCT_AXIS0));
  m.attr("DCT_1D") = py::int_(static_cast<int>(SDCT_DCT_1D));
  m.attr("IDCT_1D") = py::int_(static_cast<int>(SDCT_IDCT_1D));
  m.attr("IDXST_1D") = py::int_(static_cast<int>(SDCT_IDXST_1D));
}
