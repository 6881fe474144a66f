// ftconv_b200/checksums.hpp -- the reference's checksum and detection building blocks
// (proj/core/include/ftconv/checksums.hpp, schemes.hpp:79-94) re-exposed over the B200
// C ABI.  Host tensors in, host results out; every reduction runs on the device in the
// reference's association order at T=double, so the results are bitwise what
// ftconv::<fn><double> returns on the same FP32 data (tests/cpp/test_blocks.cpp).
//
//   kernel_checksums   checksums.hpp:70-88    -> ftc_kernel_checksums
//   input_checksums    checksums.hpp:91-113   -> ftc_input_checksums + ftc_kernel_checksums
//   output_checksums   checksums.hpp:134-161  -> ftc_output_checksums
//   output_summations  checksums.hpp:165-190  -> ftc_output_summations
//     (+ bias_adjust   checksums.hpp:195-248, fused: pass the bias)
//   values_differ / grids_consistent  checksums.hpp:54-67 (host predicates, same rule)
//   verify_kernel      checksums.hpp:250-259  -> ftc_verify_kernel
//   detect_coc_d       schemes.hpp:79-94      -> ftc_detect_coc_d
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <optional>
#include <vector>

#include "ftconv.hpp"

namespace ftconv_b200 {

/// CkSel (checksums.hpp:14-23)
enum CkSel : unsigned {
  CK_O1 = FTC_CK_O1, CK_O2 = FTC_CK_O2, CK_O3 = FTC_CK_O3, CK_O4 = FTC_CK_O4,
  CK_O5 = FTC_CK_O5, CK_O6 = FTC_CK_O6, CK_O7 = FTC_CK_O7, CK_ALL = FTC_CK_ALL
};

/// checksums.hpp:28-34
struct InputChecksums {
  Tensor4d cd1;
  std::optional<Tensor4d> cd2;
  Tensor4d cw1;
  std::optional<Tensor4d> cw2;
};

/// checksums.hpp:37-44: Co1/Co3 per column m, Co2/Co4 per row n, Co5..7 one grid.
struct OutputChecksums {
  std::optional<std::vector<Grid>> co1, co2, co3, co4;
  std::optional<Grid> co5, co6, co7;
};

/// checksums.hpp:47-51
struct OutputSummations {
  std::optional<std::vector<Grid>> so1, so2, so3, so4;
  std::optional<Grid> so5, so6, so7;
};

/// schemes.hpp:17-22
struct DetectionResult {
  bool clean = true;
  std::vector<std::uint8_t> mismatch_mask;  // E*E, row-major
  double max_rel_dev = 0.0;
};

/// values_differ (checksums.hpp:54-60): mismatch when |c-s| > tau * max(|c|,|s|,1).
inline bool values_differ(double c, double s, double tau) {
  return std::abs(c - s) > tau * std::max({std::abs(c), std::abs(s), 1.0});
}

/// grids_consistent (checksums.hpp:62-67)
inline bool grids_consistent(const Grid& c, const Grid& s, double tau) {
  for (std::size_t i = 0; i < c.v.size(); ++i)
    if (values_differ(c.v[i], s.v[i], tau)) return false;
  return true;
}

namespace detail {

/// Device allocation through the library's runtime (ftc_device_alloc): the host
/// program links only libftconv_b200.so.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    void* p = nullptr;
    check(ftc_device_alloc(n * sizeof(T), &p), "ftc_device_alloc");
    p_ = static_cast<T*>(p);
  }
  DeviceBuffer(const T* host, std::size_t n) : DeviceBuffer(n) { upload(host); }
  ~DeviceBuffer() { ftc_device_free(p_); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* host) { check(ftc_memcpy(p_, host, n_ * sizeof(T), 0, nullptr), "ftc_memcpy h2d"); }
  void download(T* host) const { check(ftc_memcpy(host, p_, n_ * sizeof(T), 1, nullptr), "ftc_memcpy d2h"); }
  std::vector<T> to_host() const {
    std::vector<T> h(n_);
    download(h.data());
    return h;
  }
  void zero() { check(ftc_memset_zero(p_, n_ * sizeof(T), nullptr), "ftc_memset_zero"); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

/// descriptor of a kernel-only call: D is a 1 x Ckw*groups x R x R probe (E = 1)
inline ftc_conv_desc kernel_desc(const Tensor4& W, std::size_t groups) {
  if (groups == 0 || W.dim(0) % groups != 0) throw ConfigError("groups must divide M");
  ftc_conv_desc d{};
  d.N = 1;
  d.C = (int32_t)(W.dim(1) * groups);
  d.H = (int32_t)W.dim(2);
  d.M = (int32_t)W.dim(0);
  d.R = (int32_t)W.dim(2);
  d.stride = 1;
  d.pad = 0;
  d.groups = (int32_t)groups;
  return d;
}

inline std::vector<Grid> split_grids(const std::vector<double>& v, std::size_t count, std::size_t E) {
  std::vector<Grid> out(count, Grid(E));
  for (std::size_t b = 0; b < count; ++b)
    std::copy(v.begin() + b * E * E, v.begin() + (b + 1) * E * E, out[b].v.begin());
  return out;
}

inline Grid one_grid(const std::vector<double>& v, std::size_t E) {
  Grid g(E);
  std::copy(v.begin(), v.begin() + E * E, g.v.begin());
  return g;
}

}  // namespace detail

/// kernel_checksums (checksums.hpp:70-88): Cw1 = sum_m W_m, Cw2 = sum_m m*W_m, both
/// (1, Ckw*groups, R, R) with the per-group sums channel-concatenated.
inline void kernel_checksums(const Tensor4& W, std::size_t groups, Tensor4d& cw1, Tensor4d& cw2) {
  const ftc_conv_desc d = detail::kernel_desc(W, groups);
  const std::size_t nCw = (std::size_t)d.C * d.R * d.R;
  detail::DeviceBuffer<float> Wd(W.data(), W.size());
  detail::DeviceBuffer<double> c1(nCw), c2(nCw);
  check(ftc_kernel_checksums(&d, Wd.get(), c1.get(), c2.get(), nullptr), "kernel_checksums");
  cw1 = Tensor4d(1, (std::size_t)d.C, d.R, d.R);
  cw2 = Tensor4d(1, (std::size_t)d.C, d.R, d.R);
  c1.download(cw1.data());
  c2.download(cw2.data());
}

/// input_checksums (checksums.hpp:91-113): Cd1 = sum_n D_n, Cd2 = sum_n n*D_n (ascending
/// n) plus the kernel checksums.
inline InputChecksums input_checksums(const Tensor4& D, const Tensor4& W, std::size_t groups) {
  if (groups == 0 || D.dim(1) % groups != 0) throw ConfigError("groups must divide Ch");
  if (W.dim(1) != D.dim(1) / groups) throw ShapeError("kernel channels must be Ch/groups");
  if (D.dim(2) != D.dim(3)) throw ShapeError("fmap must be square (H x H)");
  ftc_conv_desc d{};  // the D reduction reads no geometry: a 1x1 probe conv
  d.N = (int32_t)D.dim(0);
  d.C = (int32_t)D.dim(1);
  d.H = (int32_t)D.dim(2);
  d.M = (int32_t)W.dim(0);
  d.R = 1;
  d.stride = 1;
  d.groups = (int32_t)groups;
  const std::size_t nCd = D.dim(1) * D.dim(2) * D.dim(3);
  detail::DeviceBuffer<float> Dd(D.data(), D.size());
  detail::DeviceBuffer<double> c1(nCd), c2(nCd);
  check(ftc_input_checksums(&d, Dd.get(), c1.get(), c2.get(), nullptr), "input_checksums");
  InputChecksums ic;
  ic.cd1 = Tensor4d(1, D.dim(1), D.dim(2), D.dim(3));
  ic.cd2 = Tensor4d(1, D.dim(1), D.dim(2), D.dim(3));
  c1.download(ic.cd1.data());
  c2.download(ic.cd2->data());
  Tensor4d cw1, cw2;
  kernel_checksums(W, groups, cw1, cw2);
  ic.cw1 = std::move(cw1);
  ic.cw2 = std::move(cw2);
  return ic;
}

/// output_checksums (checksums.hpp:134-161): the convolutions of the input checksums
/// selected by `which`, each in the reference's (k, i, j) accumulation order.
inline OutputChecksums output_checksums(unsigned which, const Tensor4& D, const Tensor4& W,
                                        const InputChecksums& ic, const ConvParams& p) {
  if ((which & (CK_O3 | CK_O7)) && !ic.cd2) throw ConfigError("requested checksum needs Cd2 which is absent");
  if ((which & (CK_O4 | CK_O6)) && !ic.cw2) throw ConfigError("requested checksum needs Cw2 which is absent");
  ConvParams q = p;
  q.bias_enabled = false;
  const ftc_conv_desc d = detail::make_desc(D, W, q);
  const std::size_t E = output_extent(D.dim(2), W.dim(2), p);
  const std::size_t N = D.dim(0), M = W.dim(0), E2 = E * E;
  detail::DeviceBuffer<float> Dd(D.data(), D.size()), Wd(W.data(), W.size());
  detail::DeviceBuffer<double> cd1(ic.cd1.data(), ic.cd1.size()), cw1(ic.cw1.data(), ic.cw1.size());
  detail::DeviceBuffer<double> cd2, cw2;
  if (ic.cd2) cd2 = detail::DeviceBuffer<double>(ic.cd2->data(), ic.cd2->size());
  if (ic.cw2) cw2 = detail::DeviceBuffer<double>(ic.cw2->data(), ic.cw2->size());
  const std::size_t counts[7] = {M, N, M, N, 1, 1, 1};
  std::vector<detail::DeviceBuffer<double>> co;
  double* ptrs[7] = {nullptr};
  for (int k = 0; k < 7; ++k) {
    co.emplace_back((which >> k) & 1u ? counts[k] * E2 : 0);
    ptrs[k] = co.back().get();
  }
  check(ftc_output_checksums(&d, which, Dd.get(), Wd.get(), cd1.get(), cd2.get(), cw1.get(), cw2.get(), ptrs,
                             nullptr),
        "output_checksums");
  OutputChecksums cs;
  if (which & CK_O1) cs.co1 = detail::split_grids(co[0].to_host(), M, E);
  if (which & CK_O2) cs.co2 = detail::split_grids(co[1].to_host(), N, E);
  if (which & CK_O3) cs.co3 = detail::split_grids(co[2].to_host(), M, E);
  if (which & CK_O4) cs.co4 = detail::split_grids(co[3].to_host(), N, E);
  if (which & CK_O5) cs.co5 = detail::one_grid(co[4].to_host(), E);
  if (which & CK_O6) cs.co6 = detail::one_grid(co[5].to_host(), E);
  if (which & CK_O7) cs.co7 = detail::one_grid(co[6].to_host(), E);
  return cs;
}

/// output_summations (checksums.hpp:165-190) of O (N, M, E, E); with `bias` the
/// reference's bias_adjust (checksums.hpp:240-248, BiasAdjuster :195-238) is applied in
/// the same kernels, in the same order.
inline OutputSummations output_summations(const Tensor4& O, unsigned which, const Tensor4* bias = nullptr) {
  const std::size_t N = O.dim(0), M = O.dim(1), E = O.dim(2), E2 = E * E;
  if (O.dim(3) != E) throw ShapeError("output must be square (E x E)");
  if (bias && bias->dim(0) != M) throw ShapeError("bias length must equal M");
  detail::DeviceBuffer<float> Od(O.data(), O.size());
  detail::DeviceBuffer<float> Bd;
  if (bias) Bd = detail::DeviceBuffer<float>(bias->data(), M);
  const std::size_t counts[7] = {M, N, M, N, 1, 1, 1};
  std::vector<detail::DeviceBuffer<double>> so;
  double* ptrs[7] = {nullptr};
  for (int k = 0; k < 7; ++k) {
    so.emplace_back((which >> k) & 1u ? counts[k] * E2 : 0);
    ptrs[k] = so.back().get();
  }
  check(ftc_output_summations((int32_t)N, (int32_t)M, (int32_t)E, Od.get(), which, bias ? Bd.get() : nullptr, ptrs,
                              nullptr),
        "output_summations");
  OutputSummations s;
  if (which & CK_O1) s.so1 = detail::split_grids(so[0].to_host(), M, E);
  if (which & CK_O2) s.so2 = detail::split_grids(so[1].to_host(), N, E);
  if (which & CK_O3) s.so3 = detail::split_grids(so[2].to_host(), M, E);
  if (which & CK_O4) s.so4 = detail::split_grids(so[3].to_host(), N, E);
  if (which & CK_O5) s.so5 = detail::one_grid(so[4].to_host(), E);
  if (which & CK_O6) s.so6 = detail::one_grid(so[5].to_host(), E);
  if (which & CK_O7) s.so7 = detail::one_grid(so[6].to_host(), E);
  return s;
}

/// verify_kernel (checksums.hpp:250-259): true iff the fresh Cw1 of W matches cw1_ref.
inline bool verify_kernel(const Tensor4& W, const Tensor4d& cw1_ref, std::size_t groups, double tau) {
  const ftc_conv_desc d = detail::kernel_desc(W, groups);
  if (cw1_ref.dim(0) != 1 || cw1_ref.dim(1) != (std::size_t)d.C || cw1_ref.dim(2) != (std::size_t)d.R ||
      cw1_ref.dim(3) != (std::size_t)d.R)
    throw ShapeError("kernel checksum shape mismatch");
  detail::DeviceBuffer<float> Wd(W.data(), W.size());
  detail::DeviceBuffer<double> ref(cw1_ref.data(), cw1_ref.size());
  int32_t ok = 0;
  check(ftc_verify_kernel(&d, Wd.get(), ref.get(), tau, &ok, nullptr), "verify_kernel");
  return ok != 0;
}

/// detect_coc_d (schemes.hpp:79-94): elementwise CoC-D over the Co5/So5 grids.
inline DetectionResult detect_coc_d(const Grid& co5, const Grid& so5, double tau) {
  if (co5.v.size() != so5.v.size()) throw ShapeError("grid size mismatch");
  const std::size_t E2 = co5.v.size();
  detail::DeviceBuffer<double> c(co5.v.data(), E2), s(so5.v.data(), E2);
  detail::DeviceBuffer<std::uint8_t> mask(E2);
  int32_t clean = 1;
  DetectionResult r;
  check(ftc_detect_coc_d(c.get(), s.get(), (int32_t)E2, tau, mask.get(), &clean, &r.max_rel_dev, nullptr),
        "detect_coc_d");
  r.clean = clean != 0;
  r.mismatch_mask = mask.to_host();
  return r;
}

}  // namespace ftconv_b200
