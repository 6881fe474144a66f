// The checksum / detection building blocks (include/ftconv_b200/checksums.hpp) against
// host restatements of the reference loops at T=double (checksums.hpp:70-190,
// conv.hpp:135-145, schemes.hpp:79-94): the sums run in the reference's association
// order on both sides, so every comparison is bitwise.  Built and run by
// tests/test_gpu_cpp_api.py on the GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "ftconv_b200/checksums.hpp"

using namespace ftconv_b200;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);        \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

// conv_block (conv.hpp:135-145): [1,C,H,H] (*) [1,C,R,R] -> E x E, (k,i,j) order, FP64
static Grid conv_block_host(const Tensor4d& X, const Tensor4d& K, std::size_t U, std::size_t pad, std::size_t E) {
  const std::size_t C = X.dim(1), H = X.dim(2), R = K.dim(2);
  Grid g(E);
  for (std::size_t x = 0; x < E; ++x)
    for (std::size_t y = 0; y < E; ++y) {
      double acc = 0.0;
      for (std::size_t k = 0; k < C; ++k)
        for (std::size_t i = 0; i < R; ++i)
          for (std::size_t j = 0; j < R; ++j) {
            const long long a = (long long)(U * x + i) - (long long)pad, b = (long long)(U * y + j) - (long long)pad;
            const double v = (a < 0 || b < 0 || a >= (long long)H || b >= (long long)H) ? 0.0 : X(0, k, a, b);
            acc += v * K(0, k, i, j);
          }
      g(x, y) = acc;
    }
  return g;
}

int main() {
  const std::size_t N = 5, C = 6, H = 9, M = 7, R = 3, G = 1;
  ConvParams p;
  p.pad = 1;
  p.bias_enabled = true;
  const Tensor4 D = Tensor4::random(N, C, H, H, 71, 0.0, 1.0);
  const Tensor4 W = Tensor4::random(M, C, R, R, 72, -0.3, 0.3);
  Tensor4 B(M, 1, 1, 1);
  for (std::size_t m = 0; m < M; ++m) B(m, 0, 0, 0) = 0.05f * (float)m - 0.1f;

  // kernel_checksums (checksums.hpp:70-88)
  Tensor4d cw1, cw2;
  kernel_checksums(W, G, cw1, cw2);
  Tensor4d hw1(1, C, R, R), hw2(1, C, R, R);
  for (std::size_t m = 0; m < M; ++m)
    for (std::size_t k = 0; k < C; ++k)
      for (std::size_t i = 0; i < R; ++i)
        for (std::size_t j = 0; j < R; ++j) {
          hw1(0, k, i, j) += (double)W(m, k, i, j);
          hw2(0, k, i, j) += (double)m * (double)W(m, k, i, j);
        }
  CHECK(same_bits(cw1.raw(), hw1.raw()));
  CHECK(same_bits(cw2.raw(), hw2.raw()));

  // input_checksums (checksums.hpp:91-113)
  const InputChecksums ic = input_checksums(D, W, G);
  Tensor4d hd1(1, C, H, H), hd2(1, C, H, H);
  for (std::size_t n = 0; n < N; ++n)
    for (std::size_t k = 0; k < C; ++k)
      for (std::size_t a = 0; a < H; ++a)
        for (std::size_t b = 0; b < H; ++b) {
          hd1(0, k, a, b) += (double)D(n, k, a, b);
          hd2(0, k, a, b) += (double)n * (double)D(n, k, a, b);
        }
  CHECK(same_bits(ic.cd1.raw(), hd1.raw()));
  CHECK(ic.cd2 && same_bits(ic.cd2->raw(), hd2.raw()));
  CHECK(same_bits(ic.cw1.raw(), hw1.raw()));

  // output_checksums Co5..Co7 (checksums.hpp:157-159 -> conv_block)
  const std::size_t E = output_extent(H, R, p);
  const OutputChecksums cs = output_checksums(CK_ALL, D, W, ic, p);
  CHECK(cs.co5 && same_bits(cs.co5->v, conv_block_host(hd1, hw1, 1, 1, E).v));
  CHECK(cs.co6 && same_bits(cs.co6->v, conv_block_host(hd1, hw2, 1, 1, E).v));
  CHECK(cs.co7 && same_bits(cs.co7->v, conv_block_host(hd2, hw1, 1, 1, E).v));
  CHECK(cs.co1 && cs.co1->size() == M && cs.co2 && cs.co2->size() == N);
  CHECK(cs.co3 && cs.co3->size() == M && cs.co4 && cs.co4->size() == N);
  {  // ConfigError when a requested family lacks its input (checksums.hpp:139-142)
    InputChecksums partial = ic;
    partial.cd2.reset();
    bool threw = false;
    try {
      output_checksums(CK_O7, D, W, partial, p);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }

  // output_summations + bias_adjust (checksums.hpp:165-248) on the device conv's output
  const Tensor4 O = conv_forward(D, W, &B, p);
  const OutputSummations so = output_summations(O, CK_ALL, &B);
  Grid h5(E), h6(E), h7(E);
  for (std::size_t n = 0; n < N; ++n)
    for (std::size_t m = 0; m < M; ++m)
      for (std::size_t x = 0; x < E; ++x)
        for (std::size_t y = 0; y < E; ++y) {
          const double v = (double)O(n, m, x, y);
          h5(x, y) += v;
          h6(x, y) += (double)m * v;
          h7(x, y) += (double)n * v;
        }
  double sum_b = 0.0, sum_mb = 0.0;
  for (std::size_t m = 0; m < M; ++m) {
    sum_b += (double)B(m, 0, 0, 0);
    sum_mb += (double)m * (double)B(m, 0, 0, 0);
  }
  const double nN = (double)N, wn = (double)(N * (N - 1) / 2);
  for (double& v : h5.v) v -= nN * sum_b;
  for (double& v : h6.v) v -= nN * sum_mb;
  for (double& v : h7.v) v -= wn * sum_b;
  CHECK(so.so5 && same_bits(so.so5->v, h5.v));
  CHECK(so.so6 && same_bits(so.so6->v, h6.v));
  CHECK(so.so7 && same_bits(so.so7->v, h7.v));
  CHECK(so.so1 && so.so1->size() == M && so.so2 && so.so2->size() == N);

  // the FP32 conv is consistent with its checksums; values_differ / grids_consistent
  CHECK(grids_consistent(*cs.co5, *so.so5, 1e-5));
  CHECK(grids_consistent(*cs.co6, *so.so6, 1e-5));
  CHECK(grids_consistent(*cs.co7, *so.so7, 1e-5));
  for (std::size_t m = 0; m < M; ++m) CHECK(grids_consistent((*cs.co1)[m], (*so.so1)[m], 1e-5));
  for (std::size_t n = 0; n < N; ++n) CHECK(grids_consistent((*cs.co2)[n], (*so.so2)[n], 1e-5));
  CHECK(!values_differ(100.0, 100.0 + 1e-4, 1e-5) && values_differ(100.0, 100.01, 1e-5));
  CHECK(!values_differ(0.0, 5e-6, 1e-5) && values_differ(0.0, 2e-5, 1e-5));

  // detect_coc_d (schemes.hpp:79-94): clean, then one corrupted position
  DetectionResult clean = detect_coc_d(*cs.co5, *so.so5, 1e-5);
  CHECK(clean.clean && clean.mismatch_mask.size() == E * E);
  double mrd = 0.0;
  for (std::size_t i = 0; i < E * E; ++i) {
    const double c = cs.co5->v[i], s = so.so5->v[i];
    mrd = std::max(mrd, std::abs(c - s) / std::max({std::abs(c), std::abs(s), 1.0}));
  }
  CHECK(clean.max_rel_dev == mrd);
  Grid bad = *so.so5;
  bad(3, 4) += 1.0;
  DetectionResult dirty = detect_coc_d(*cs.co5, bad, 1e-5);
  CHECK(!dirty.clean);
  for (std::size_t i = 0; i < E * E; ++i) CHECK(dirty.mismatch_mask[i] == (i == 3 * E + 4 ? 1 : 0));

  // verify_kernel (checksums.hpp:250-259): golden W passes, a corrupted W does not
  CHECK(verify_kernel(W, cw1, G, 1e-5));
  Tensor4 Wbad = W;
  Wbad(2, 1, 0, 2) += 0.5f;
  CHECK(!verify_kernel(Wbad, cw1, G, 1e-5));
  {
    bool threw = false;
    try {
      verify_kernel(W, Tensor4d(1, C + 1, R, R), G, 1e-5);
    } catch (const ShapeError&) {
      threw = true;
    }
    CHECK(threw);
  }

  // grouped kernel checksums: per-group sums channel-concatenated (checksums.hpp:76-87)
  {
    const std::size_t g2 = 2, Mg = 4, Ckw = 3;
    const Tensor4 Wg = Tensor4::random(Mg, Ckw, R, R, 73);
    Tensor4d a, b;
    kernel_checksums(Wg, g2, a, b);
    Tensor4d ha(1, Ckw * g2, R, R), hb(1, Ckw * g2, R, R);
    for (std::size_t g = 0; g < g2; ++g)
      for (std::size_t mg = 0; mg < Mg / g2; ++mg) {
        const std::size_t m = g * (Mg / g2) + mg;
        for (std::size_t k = 0; k < Ckw; ++k)
          for (std::size_t i = 0; i < R; ++i)
            for (std::size_t j = 0; j < R; ++j) {
              ha(0, g * Ckw + k, i, j) += (double)Wg(m, k, i, j);
              hb(0, g * Ckw + k, i, j) += (double)m * (double)Wg(m, k, i, j);
            }
      }
    CHECK(same_bits(a.raw(), ha.raw()) && same_bits(b.raw(), hb.raw()));
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
