// C++ drop-in check: a program written against the reference's operator API
// (proj/include/sdct: Plan2d, dct_2d, idct_2d, idct_idxst_2d, Plan3d, dct_3d,
// force_demo_fields, StageCounters, the exception types) compiled against
// include/sdct and linked with libsdct_b200.so instead of sdct_core.
// Prints one line per check; exit code 0 when every check passes.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "sdct/dct2d.hpp"
#include "sdct/errors.hpp"
#include "sdct/force.hpp"
#include "sdct/transforms_ext.hpp"

namespace {

sdct::RealTensor random_tensor(const sdct::Shape& shape, unsigned seed) {
  std::mt19937 rng(seed);  // proj/tests/test_dct2d.cpp:17-23
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  sdct::RealTensor t(shape);
  for (std::size_t i = 0; i < t.size(); ++i) t[i] = u(rng);
  return t;
}

double rel_l2(const sdct::RealTensor& a, const sdct::RealTensor& b, double scale = 1.0) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double d = a[i] * scale - b[i];
    num += d * d;
    den += b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

int failures = 0;
void check(bool ok, const char* what, double v) {
  std::printf("%s %s (%.3e)\n", ok ? "PASS" : "FAIL", what, v);
  if (!ok) ++failures;
}

}  // namespace

int main() {
  try {
    // 2D round trip through a reused plan: idct_2d(dct_2d(x)) == N1 N2 / 4 x
    const sdct::RealTensor x = random_tensor(sdct::Shape{256, 512}, 7);
    const sdct::Plan2d plan(256, 512);
    const sdct::RealTensor y = sdct::dct_2d(x, plan);
    const sdct::RealTensor z = sdct::idct_2d(y, plan);
    const double e = rel_l2(z, x, 4.0 / (256.0 * 512.0));
    check(e < 1e-13, "2D round trip 256x512", e);

    // known answer: 2x2 ones -> [[4,0],[0,0]]
    sdct::RealTensor ones(sdct::Shape{2, 2});
    for (std::size_t i = 0; i < 4; ++i) ones[i] = 1.0;
    const sdct::RealTensor k = sdct::dct_2d(ones);
    check(std::fabs(k[0] - 4.0) < 1e-12 && std::fabs(k[1]) + std::fabs(k[2]) + std::fabs(k[3]) < 1e-12,
          "2x2 ones known answer", k[0]);

    // column-0-only input is annihilated by idct_idxst_2d (test_transforms_ext.cpp:158-170)
    sdct::RealTensor c0(sdct::Shape{8, 8});
    for (std::size_t i = 0; i < 8; ++i) c0[i * 8] = 1.0 + static_cast<double>(i);
    const sdct::RealTensor w = sdct::idct_idxst_2d(c0, sdct::Plan2d(8, 8));
    double mx = 0.0;
    for (std::size_t i = 0; i < w.size(); ++i) mx = std::fmax(mx, std::fabs(w[i]));
    check(mx < 1e-12, "idct_idxst_2d annihilates column 0", mx);

    // 3D round trip: idct_3d(dct_3d(x)) == N1 N2 N3 / 8 x
    const sdct::RealTensor x3 = random_tensor(sdct::Shape{16, 8, 32}, 9);
    const sdct::RealTensor z3 = sdct::idct_3d(sdct::dct_3d(x3));
    const double e3 = rel_l2(z3, x3, 8.0 / (16.0 * 8.0 * 32.0));
    check(e3 < 1e-13, "3D round trip 16x8x32", e3);

    // counters of one 8x8 dct_2d: 360 mults / 260 adds (test_dct2d.cpp:246-258)
    sdct::StageCounters cnt;
    sdct::dct_2d(random_tensor(sdct::Shape{8, 8}, 3), sdct::Plan2d(8, 8), {}, &cnt);
    check(cnt.real_mults == 360 && cnt.real_adds == 260, "8x8 counters 360/260",
          static_cast<double>(cnt.real_mults));

    // force fields are finite and vanish for a constant density (only DC survives)
    sdct::RealTensor flat(sdct::Shape{32, 32});
    for (std::size_t i = 0; i < flat.size(); ++i) flat[i] = 0.5;
    const sdct::ForceFields f = sdct::force_demo_fields(flat);
    double fm = 0.0;
    for (std::size_t i = 0; i < f.xi1.size(); ++i) fm = std::fmax(fm, std::fabs(f.xi1[i]) + std::fabs(f.xi2[i]));
    check(fm < 1e-9, "force fields of a constant density", fm);

    // concurrent host calls (the reference's calls are reentrant):
    // four threads sharing one plan and four with their own plans, fast and
    // generic shapes, agree bit for bit with serial results
    {
      const sdct::RealTensor xa = random_tensor(sdct::Shape{512, 256}, 21);
      const sdct::RealTensor xb = random_tensor(sdct::Shape{300, 200}, 22);
      const sdct::Plan2d shared(512, 256);
      const sdct::RealTensor ya = sdct::dct_2d(xa, shared);
      const sdct::RealTensor yb = sdct::idct_2d(xb, sdct::Plan2d(300, 200));
      std::atomic<int> bad{0};
      std::vector<std::thread> ts;
      for (int i = 0; i < 8; ++i)
        ts.emplace_back([&, i] {
          for (int r = 0; r < 5; ++r) {
            if (i < 4) {
              const sdct::RealTensor o = sdct::dct_2d(xa, shared);
              if (o.storage() != ya.storage()) ++bad;
            } else {
              const sdct::RealTensor o = sdct::idct_2d(xb, sdct::Plan2d(300, 200));
              if (o.storage() != yb.storage()) ++bad;
            }
          }
        });
      for (auto& th : ts) th.join();
      check(bad.load() == 0, "8 threads x 5 calls (shared + private plans) match serial", bad.load());
    }

    // errors keep the reference's types (proj/include/sdct/errors.hpp:11-33)
    bool threw = false;
    try {
      sdct::dct_2d(x3);
    } catch (const sdct::ShapeError&) {
      threw = true;
    }
    check(threw, "rank mismatch throws ShapeError", 0.0);
  } catch (const std::exception& ex) {
    std::printf("FAIL exception: %s\n", ex.what());
    return 2;
  }
  return failures ? 1 : 0;
}
