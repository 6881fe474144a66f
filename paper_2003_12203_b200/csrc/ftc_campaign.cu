// ftc_campaign.cu -- fault campaigns: corpus generation, ground truth and the mapping of a
// FaultSpec onto the device fault records (fault.hpp:42-291).
//
// Host code.  The corpus must be bit-identical to the reference's, so it draws from the
// same standard-library generator and distributions (std::mt19937_64,
// std::discrete_distribution, std::uniform_real_distribution<double>) in the same order;
// the reference is header-only C++ on the same toolchain, so the draws coincide.
#include <cstdint>
#include <random>

#include "ftc_common.cuh"

namespace {

enum SpecTarget { kOutBlock = 0, kOutRow, kOutCol, kFmap, kKernel, kChecksum };
enum SpecChecksum { kCkNone = 0, kCd1, kCd2, kCw1, kCw2 };

void truth_of(const ftc_fault_spec& f, int64_t N, int64_t M, ftc_ground_truth* g) {
  g->benign = 0;
  g->output_diverges = 0;
  g->expected_stage = FTC_STAGE_NONE;
  switch (f.target) {
    case kOutBlock:  // one block: CoC locates it
      g->expected_stage = FTC_STAGE_COC;
      break;
    case kOutRow:  // a block row: RC (a single column of blocks degenerates to one block)
      g->expected_stage = M == 1 ? FTC_STAGE_COC : FTC_STAGE_RC;
      break;
    case kOutCol:
      g->expected_stage = N == 1 ? FTC_STAGE_COC : FTC_STAGE_CLC;
      break;
    case kFmap:  // a corrupted input map corrupts its output row; n = 0 looks like Cd corruption
      if (M == 1) {
        g->expected_stage = FTC_STAGE_COC;
      } else if (f.i == 0) {
        g->expected_stage = FTC_STAGE_DISCARD;
        g->output_diverges = 1;
      } else {
        g->expected_stage = FTC_STAGE_RC;
      }
      break;
    case kKernel:  // a corrupted kernel corrupts its output column
      g->expected_stage = N == 1 ? FTC_STAGE_COC : FTC_STAGE_CLC;
      break;
    case kChecksum:
      if (f.checksum == kCd1) {
        g->expected_stage = FTC_STAGE_DISCARD;
      } else if (f.checksum == kCw1) {
        g->expected_stage = FTC_STAGE_RELOAD;
      } else {  // cd2 / cw2 feed no detection-path checksum
        g->benign = 1;
        g->expected_stage = FTC_STAGE_NONE;
      }
      break;
  }
}

}  // namespace

extern "C" {

int ftc_ground_truth_of(const ftc_fault_spec* spec, int64_t N, int64_t M, ftc_ground_truth* out) {
  if (!spec || !out) {
    ftc::set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  truth_of(*spec, N, M, out);
  return FTC_OK;
}

int ftc_campaign(const ftc_layer_grid* layers, int32_t n_layers, int64_t n_runs, const double* weights6,
                 uint64_t seed, ftc_fault_spec* specs, ftc_ground_truth* truths) {
  if (!layers || n_layers <= 0) {
    ftc::set_error(FTC_CONFIG_ERROR, "campaign needs at least one layer");
    return FTC_CONFIG_ERROR;
  }
  if (!weights6 || !specs || n_runs < 0) {
    ftc::set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  for (int k = 0; k < 6; ++k)
    if (weights6[k] < 0) {
      ftc::set_error(FTC_CONFIG_ERROR, "target weights must be nonnegative");
      return FTC_CONFIG_ERROR;
    }
  std::mt19937_64 rng(seed);
  std::discrete_distribution<int> target_of(weights6, weights6 + 6);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  // an index in [0, n): floor(u * n), folded back in case u * n rounds up to n
  auto pick = [&](int64_t n) { return (int64_t)((uint64_t)(unit(rng) * (double)n) % (uint64_t)n); };
  for (int64_t r = 0; r < n_runs; ++r) {
    const ftc_layer_grid& g = layers[r % n_layers];
    ftc_fault_spec f{};
    f.layer_index = (int32_t)(r % n_layers);
    f.target = target_of(rng);
    f.seed = rng();
    f.i = pick(g.N);
    f.j = pick(g.M);
    f.x = f.y = -1;
    f.mode = 0;  // additive perturbation
    f.bit = 23;
    const bool single = unit(rng) < 0.5;
    if (f.target == kChecksum) {
      static const int names[4] = {kCd1, kCd2, kCw1, kCw2};
      f.checksum = names[pick(4)];
      const int64_t side = (f.checksum == kCw1 || f.checksum == kCw2) ? g.R : g.H;
      f.x = pick(side);
      f.y = pick(side);
    } else if (f.target == kFmap) {
      if (single) {
        f.x = pick(g.H);
        f.y = pick(g.H);
      }
    } else if (f.target == kKernel) {
      if (single) {
        f.x = pick(g.R);
        f.y = pick(g.R);
      }
    } else {
      const int64_t E = g.H - g.R + 1;  // campaign layers: stride 1, no padding
      if (single) {
        f.x = pick(E);
        f.y = pick(E);
      }
    }
    // bit flips only on single-element output-block faults, every 7th run
    if (f.target == kOutBlock && f.x >= 0 && r % 7 == 3) {
      f.mode = 1;
      f.bit = 23;
    }
    specs[r] = f;
    if (truths) truth_of(f, g.N, g.M, &truths[r]);
  }
  return FTC_OK;
}

int ftc_spec_faults(const ftc_fault_spec* spec, ftc_fault* out, int32_t* n_out) {
  if (!spec || !out || !n_out) {
    ftc::set_error(FTC_INVALID_ARGUMENT, "null argument");
    return FTC_INVALID_ARGUMENT;
  }
  const ftc_fault_spec& f = *spec;
  ftc_fault d{};
  d.mode = f.mode == 1 ? FTC_FAULT_BITFLIP : FTC_FAULT_SCALE;
  d.bit = f.bit;
  d.seed = f.seed;
  const bool all = f.x < 0;
  switch (f.target) {
    case kOutBlock: case kOutRow: case kOutCol:
      d.target = FTC_FAULT_OUTPUT;
      d.n = f.target == kOutCol ? -1 : (int32_t)f.i;
      d.m = f.target == kOutRow ? -1 : (int32_t)f.j;
      d.x = all ? -1 : (int32_t)f.x;
      d.y = all ? -1 : (int32_t)f.y;
      break;
    case kFmap: case kKernel: case kChecksum:
      // hit_tensor: one element (block, channel 0, x, y), or the whole block
      if (f.target == kFmap) {
        d.target = FTC_FAULT_FMAP;
        d.n = (int32_t)f.i;
      } else if (f.target == kKernel) {
        d.target = FTC_FAULT_KERNEL;
        d.n = (int32_t)f.j;
      } else {
        switch (f.checksum) {
          case kCd1: d.target = FTC_FAULT_CD1; break;
          case kCd2: d.target = FTC_FAULT_CD2; break;
          case kCw1: d.target = FTC_FAULT_CW1; break;
          case kCw2: d.target = FTC_FAULT_CW2; break;
          default:
            ftc::set_error(FTC_CONFIG_ERROR, "checksum fault needs a checksum name");
            return FTC_CONFIG_ERROR;
        }
        d.n = 0;
      }
      d.m = all ? -1 : 0;
      d.x = all ? -1 : (int32_t)f.x;
      d.y = all ? -1 : (int32_t)f.y;
      break;
    default:
      ftc::set_error(FTC_CONFIG_ERROR, "unknown fault target");
      return FTC_CONFIG_ERROR;
  }
  out[0] = d;
  *n_out = 1;
  return FTC_OK;
}

}  // extern "C"
