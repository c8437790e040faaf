// mdreduce_b200.hpp — drop-in C++ operator API of the B200 hot path.
//
// A reference caller (namespace mdreduce, /root/reference/proj/include/
// mdreduce/{half,mma,reduce,simblock,docking,rng,instance_io,errors}.hpp)
// includes this single header instead and links libmdr_b200.so.  Types keep
// the reference's names, members and defaults; functions keep their
// signatures and throw the same exception types before doing any work.
// Every numeric entry point runs on the GPU through the C-ABI (mdr.h); there
// is no CPU fallback.  Extensions (batched calls, the split-precision method,
// device selection) live in mdreduce::b200.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <memory>
#include <vector>

namespace mdreduce {

// ---------------------------------------------------------------- errors
// errors.hpp:10-42
class SizeError : public std::invalid_argument {
 public:
  explicit SizeError(const std::string& w) : std::invalid_argument(w) {}
};
class UnsupportedBlockSizeError : public std::invalid_argument {
 public:
  explicit UnsupportedBlockSizeError(const std::string& w) : std::invalid_argument(w) {}
};
class NumericDomainError : public std::domain_error {
 public:
  explicit NumericDomainError(const std::string& w) : std::domain_error(w) {}
};
class ParseError : public std::runtime_error {
 public:
  ParseError(int line, const std::string& what)
      : std::runtime_error(line > 0 ? "line " + std::to_string(line) + ": " + what : what), line_(line) {}
  int line() const { return line_; }

 private:
  int line_;
};
// Device / driver failure (no reference counterpart).
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------- half
// half.hpp:11-49
class Half {
 public:
  constexpr Half() : bits_(0) {}
  static constexpr Half from_bits(std::uint16_t b) {
    Half h;
    h.bits_ = b;
    return h;
  }
  constexpr std::uint16_t bits() const { return bits_; }
  friend constexpr bool operator==(Half a, Half b) { return a.bits_ == b.bits_; }
  friend constexpr bool operator!=(Half a, Half b) { return a.bits_ != b.bits_; }

 private:
  std::uint16_t bits_;
};
Half f32_to_half(float v);
float half_to_f32(Half h);
Half half_add(Half a, Half b);
inline constexpr std::uint16_t kHalfPosInf = 0x7C00;
inline constexpr std::uint16_t kHalfNegInf = 0xFC00;
inline constexpr std::uint16_t kHalfQuietNan = 0x7E00;
inline bool half_is_finite(Half h) { return (h.bits() & 0x7C00) != 0x7C00; }
inline bool half_is_nan(Half h) { return (h.bits() & 0x7C00) == 0x7C00 && (h.bits() & 0x03FF) != 0; }

// ---------------------------------------------------------------- mma
// mma.hpp:13-73
enum class Layout { RowMajor, ColMajor };
enum class AccumMode { Half, Single };

class Mat16 {
 public:
  static constexpr int kDim = 16;
  static constexpr std::size_t kElems = 256;
  Mat16() : layout_(Layout::RowMajor) { e_.fill(Half()); }
  Half at(int r, int c) const { return e_[static_cast<std::size_t>(r * kDim + c)]; }
  void set(int r, int c, Half v) { e_[static_cast<std::size_t>(r * kDim + c)] = v; }
  Layout layout() const { return layout_; }
  void set_layout(Layout l) { layout_ = l; }
  const Half* data() const { return e_.data(); }

 private:
  std::array<Half, kElems> e_;
  Layout layout_;
};

class Accum16 {
 public:
  explicit Accum16(AccumMode mode) : mode_(mode) { v_.fill(0.0f); }
  static Accum16 zero(AccumMode mode) { return Accum16(mode); }
  AccumMode mode() const { return mode_; }
  float at(int r, int c) const { return v_[static_cast<std::size_t>(r * Mat16::kDim + c)]; }
  void set(int r, int c, float v) { v_[static_cast<std::size_t>(r * Mat16::kDim + c)] = v; }
  const float* data() const { return v_.data(); }

 private:
  std::array<float, Mat16::kElems> v_;
  AccumMode mode_;
};

Mat16 load_matrix(std::span<const Half> src, Layout layout);
std::vector<float> store_matrix(const Accum16& acc, Layout layout);
Accum16 mma(const Mat16& a, const Mat16& b, const Accum16& c);

// ---------------------------------------------------------------- reduce
// reduce.hpp:13-102
enum class ReduceMethod { Baseline, Tcu, TcuSplit /* new: tf32 hi/lo MMA */ };

struct Vec4 {
  float x = 0.0f, y = 0.0f, z = 0.0f, e = 0.0f;
};
struct Partial7 {
  float e = 0.0f;
  float gx = 0.0f, gy = 0.0f, gz = 0.0f;
  float tx = 0.0f, ty = 0.0f, tz = 0.0f;
};
struct SyncStats {
  std::uint64_t block_syncs = 0;
  std::uint64_t warp_shuffles = 0;
  std::uint64_t atomic_adds = 0;
  std::uint64_t memory_fences = 0;
  std::uint64_t mma_ops = 0;
  std::uint64_t shared_mem_bytes = 0;
  std::uint64_t precision_conversions = 0;
  SyncStats& operator+=(const SyncStats& o) {
    block_syncs += o.block_syncs;
    warp_shuffles += o.warp_shuffles;
    atomic_adds += o.atomic_adds;
    memory_fences += o.memory_fences;
    mma_ops += o.mma_ops;
    shared_mem_bytes += o.shared_mem_bytes;
    precision_conversions += o.precision_conversions;
    return *this;
  }
  friend SyncStats operator+(SyncStats a, const SyncStats& b) { return a += b; }
  friend bool operator==(const SyncStats&, const SyncStats&) = default;
};

Mat16 make_p();
Mat16 make_q();
Mat16 pack_vectors(std::span<const Vec4> vs);
std::pair<Vec4, SyncStats> reduce4(std::span<const Vec4> vs, AccumMode mode);
std::pair<float, SyncStats> baseline_warp_reduce(std::span<const float> lanes);
std::pair<float, SyncStats> baseline_block_reduce(std::span<const float> values, int threads_per_block);
std::pair<std::array<float, 7>, SyncStats> reduce7(std::span<const Partial7> records, ReduceMethod method,
                                                   AccumMode accum_mode);

// ---------------------------------------------------------------- simblock
// simblock.hpp:10-65.  The reductions run on the GPU; the abstract cost
// model (estimate_cost / scaling_sweep) is kept for API compatibility and
// evaluates the same model counters the reference does (real device
// behaviour: ncu, profiles/).
struct BlockConfig {
  BlockConfig(int threads, ReduceMethod m, AccumMode a);
  int threads_per_block;
  ReduceMethod method;
  AccumMode accum_mode;
};
struct CostWeights {
  double block_sync = 10.0;
  double atomic = 4.0;
  double shuffle = 1.0;
  double fence = 4.0;
  double mma = 8.0;
};
// One block of cfg.threads_per_block records through the configured method.
std::pair<Vec4, SyncStats> simulate_block(const BlockConfig& cfg, std::span<const Vec4> values);
std::pair<std::array<float, 7>, SyncStats> simulate_block(const BlockConfig& cfg, std::span<const Partial7> values);
double estimate_cost(const SyncStats& stats, const CostWeights& weights);
struct SweepRow {
  int threads_per_block = 0;
  SyncStats baseline;
  SyncStats tcu;
  double cost_baseline = 0.0;
  double cost_tcu = 0.0;
  double cost_ratio = 0.0;  // baseline / tcu
  bool degenerate = false;  // tcu cost 0: ratio reported as 1.0
};
std::vector<SweepRow> scaling_sweep(std::span<const int> sizes, const CostWeights& weights,
                                    AccumMode accum_mode = AccumMode::Half);
inline constexpr std::array<int, 5> kDefaultSweepSizes = {64, 128, 256, 512, 1024};

// ---------------------------------------------------------------- rng
// rng.hpp:10-43 (pure uint64 arithmetic; host side)
class RngStream {
 public:
  RngStream(std::uint64_t seed, std::string_view label);
  std::uint64_t next_u64();
  double next_double();
  double uniform(double lo, double hi);
  double normal();
  std::uint64_t next_index(std::uint64_t n);

 private:
  std::uint64_t key_;
  std::uint64_t counter_ = 0;
};
inline RngStream derive_rng(std::uint64_t seed, std::string_view label) { return RngStream(seed, label); }

// ---------------------------------------------------------------- instances
// instance_io.hpp:13-49 (host I/O)
struct Atom {
  std::array<double, 3> pos{};
  double weight = 1.0;
  int torsion = -1;
};
struct Site {
  std::array<double, 3> pos{};
  double depth = 1.0;
  double preferred_distance = 1.0;
};
struct LigandInstance {
  std::vector<Atom> atoms;
  std::vector<Site> sites;
  int n_rot = 0;
  std::string name;
};
LigandInstance parse_instance(std::string_view text);
std::string serialize_instance(const LigandInstance& instance);
// One docking-run record of the results CSV (instance_io.hpp:52-65).
struct ResultRow {
  std::uint64_t seed = 0;
  std::string method;      // "baseline" | "tcu"
  std::string accum_mode;  // "half" | "single"
  std::string instance;
  double best_energy = 0.0;
  std::int64_t evaluations = 0;
  bool converged = false;
  std::uint64_t block_syncs = 0;
  std::uint64_t atomic_adds = 0;
  std::uint64_t mma_ops = 0;
  friend bool operator==(const ResultRow&, const ResultRow&) = default;
};
// RFC-4180-style CSV with the fixed header row, %.17g numbers
// (instance_io.hpp:67-73); parse_results throws ParseError(line).
std::string write_results(std::span<const ResultRow> rows);
std::vector<ResultRow> parse_results(std::string_view csv);

// ---------------------------------------------------------------- docking
// docking.hpp:17-169
struct Genotype {
  double x = 0.0, y = 0.0, z = 0.0;
  double phi = 0.0, theta = 0.0, alpha = 0.0;
  std::vector<double> torsions;
  int dim() const { return 6 + static_cast<int>(torsions.size()); }
  double get(int i) const;
  void set(int i, double v);
  void normalize_angles();
  friend bool operator==(const Genotype&, const Genotype&) = default;
};

std::array<double, 3> torsion_axis(int k);

struct ScoreResult {
  float energy = 0.0f;
  std::vector<float> gradient;
  std::array<float, 3> torque{};
  SyncStats reduce_stats;
};
ScoreResult score(const LigandInstance& instance, const Genotype& g, ReduceMethod method, AccumMode accum_mode,
                  int partition);

struct RefScore {
  double energy = 0.0;
  std::vector<double> gradient;
  std::array<double, 3> torque{};
};
RefScore score_reference(const LigandInstance& instance, const Genotype& g);

struct AdadeltaState {
  std::vector<double> avg_sq_grad;
  std::vector<double> avg_sq_update;
  double rho = 0.95;
  double epsilon = 1e-6;
  static AdadeltaState fresh(int dim, double rho = 0.95, double epsilon = 1e-6);
};
std::pair<AdadeltaState, Genotype> adadelta_step(const AdadeltaState& state, const Genotype& g,
                                                 const std::vector<double>& grad);

struct LocalSearchResult {
  Genotype genotype;
  double energy = 0.0;
  int iterations = 0;
  bool converged = false;
  SyncStats stats;
  friend bool operator==(const LocalSearchResult&, const LocalSearchResult&) = default;
};
LocalSearchResult local_search(const LigandInstance& instance, const Genotype& start, int max_iters,
                               double convergence_tol, ReduceMethod method, AccumMode accum_mode, int partition,
                               std::uint64_t rng_seed);

struct LgaSettings {
  int population_size = 36;
  int generations = 20;
  std::int64_t max_evaluations = 100000;
  double ls_fraction = 0.25;
  int ls_max_iters = 150;
  double ls_convergence_tol = 1e-4;
  double mutation_sigma = 0.3;
  int partition = 64;
};
struct LsRunRecord {
  double best_energy = 0.0;
  int iterations = 0;
  bool converged = false;
  friend bool operator==(const LsRunRecord&, const LsRunRecord&) = default;
};
struct DockResult {
  double best_energy = 0.0;
  Genotype best_genotype;
  std::int64_t evaluations = 0;
  bool converged = false;
  std::vector<LsRunRecord> runs;
  SyncStats total_stats;
  friend bool operator==(const DockResult&, const DockResult&) = default;
};
DockResult lga_run(const LigandInstance& instance, ReduceMethod method, AccumMode accum_mode,
                   const LgaSettings& settings, std::uint64_t seed);

struct MethodSummary {
  double min = 0.0, q1 = 0.0, median = 0.0, q3 = 0.0, max = 0.0;
  double mean = 0.0;
  double nonconvergent_fraction = 0.0;
};
struct ValidationReport {
  MethodSummary ref;
  MethodSummary test;
  double abs_diff_means = 0.0;
  double relative_error = 0.0;
  int n_runs = 0;
};
ValidationReport validate_pair(const LigandInstance& instance, ReduceMethod ref_method, ReduceMethod test_method,
                               AccumMode accum_mode, int n_runs, std::uint64_t base_seed,
                               const LgaSettings& settings);

// ---------------------------------------------------------------- B200 extensions
namespace b200 {
// Select the GPU used by the calls above (default 0); one context per thread.
void set_device(int device);
// Pair-term arithmetic of score / local_search / lga_run (per thread):
//   Reference — FP64 in the reference's exact operation order with
//               correctly rounded trig (399/400 paired LGA runs identical);
//   Fast64    — FP64 with FMA and one reciprocal per pair (default; float
//               outputs bit-identical to the reference on every measured
//               evaluation and local search, 382/400 paired LGA runs,
//               profiles/r2_rcp_parity.json);
//   Fp32      — FP32 pair terms: per evaluation within 1e-5 relative, but LGA
//               trajectories diverge from the reference and C3's paired-seed
//               means miss the reference's 0.2 % gate (6.7e-3): statistical
//               parity only, not for reference reproduction.
enum class PairMode { Reference, Fast64, Fp32 };
void set_pair_mode(PairMode mode);
// Torsion gradient of the analytic path (per thread; see mdr_ctx_set_exact_torsion):
// false (default) = score()'s total-torque projection, the parity quantity;
// true = exact per-group torque, the gradient score_reference() computes.
void set_exact_torsion(bool on);
// Many independent evaluations / searches / docking runs in one launch.
std::vector<ScoreResult> score_batch(const LigandInstance& instance, const std::vector<Genotype>& poses,
                                     ReduceMethod method, AccumMode accum_mode, int partition);
std::vector<LocalSearchResult> local_search_batch(const LigandInstance& instance, const std::vector<Genotype>& starts,
                                                  int max_iters, double convergence_tol, ReduceMethod method,
                                                  AccumMode accum_mode, int partition);
std::vector<DockResult> lga_run_batch(const LigandInstance& instance, ReduceMethod method, AccumMode accum_mode,
                                      const LgaSettings& settings, const std::vector<std::uint64_t>& seeds);

// ---- grid-map scoring mode (formulas in include/mdr.h) -------
struct GridShape {
  int nx = 2, ny = 2, nz = 2, n_types = 1;
  std::array<double, 3> origin{0.0, 0.0, 0.0};
  double spacing = 0.375;
};
// Maps (n_types + 2) x nz x ny x nx, x fastest: type maps, elec, desolv.
struct GridMaps {
  GridShape shape;
  std::vector<float> maps;
};
// Synthetic receptor chemistry for the map builder (mdr_receptor_fields).
struct ReceptorFields {
  std::vector<double> site_charge, site_volume, type_depth_scale, type_dist_scale;
  double elec_scale = 83.0;
  double desolv_sigma = 3.6;
};
// Per-atom ligand chemistry (mdr_ligand_params).
struct LigandChemistry {
  std::vector<int> atom_type;
  std::vector<double> charge, radius, epsilon;
  double elec_scale = 83.0;
  bool intra = true;
};
// A device-resident receptor (maps uploaded once, shared by every ligand).
class Receptor {
 public:
  static Receptor upload(const GridMaps& maps);
  // maps computed on the device from the sites of `sites`
  static Receptor build(const LigandInstance& sites, const ReceptorFields& fields, const GridShape& shape);
  GridMaps download() const;
  const GridShape& shape() const { return shape_; }
  void* handle() const { return handle_.get(); }

 private:
  GridShape shape_;
  std::shared_ptr<void> handle_;
};
// Energy, exact gradient (per-group torsion torque), inter torque per pose;
// reduce_stats are zero (no reference model counters for this mode).
std::vector<ScoreResult> grid_score_batch(const Receptor& receptor, const LigandInstance& ligand,
                                          const LigandChemistry& chem, const std::vector<Genotype>& poses,
                                          ReduceMethod method, int partition);
std::vector<LocalSearchResult> grid_local_search_batch(const Receptor& receptor, const LigandInstance& ligand,
                                                       const LigandChemistry& chem,
                                                       const std::vector<Genotype>& starts, int max_iters,
                                                       double convergence_tol, ReduceMethod method, int partition);
std::vector<DockResult> grid_lga_run_batch(const Receptor& receptor, const LigandInstance& ligand,
                                           const LigandChemistry& chem, ReduceMethod method,
                                           const LgaSettings& settings, const std::vector<std::uint64_t>& seeds);

// ---- RMSD clustering ----------------------------------------
struct Clustering {
  std::vector<int> cluster_of;        // cluster index per pose (0 = best pose's)
  std::vector<double> rmsd_to_seed;   // RMSD to the cluster's lowest-energy pose
  int n_clusters = 0;
};
std::vector<std::array<double, 3>> pose_coordinates(const LigandInstance& ligand, const Genotype& pose);
Clustering cluster_poses(const LigandInstance& ligand, const std::vector<Genotype>& poses,
                         const std::vector<double>& energies, double rmsd_tol);

// ---- virtual screen ------------------------------------------
struct ScreenResult {
  std::vector<double> best_energy;
  std::vector<Genotype> best_genotype;
  std::vector<std::int64_t> evaluations;
  std::vector<bool> converged;
  Clustering clusters;
};
// Every ligand docked runs_per_ligand times (seeds[j * runs + k]) in one
// launch sequence, then its best poses clustered.
std::vector<ScreenResult> screen_batch(const Receptor& receptor, const std::vector<LigandInstance>& ligands,
                                       const std::vector<LigandChemistry>& chemistry, int runs_per_ligand,
                                       ReduceMethod method, const LgaSettings& settings,
                                       const std::vector<std::uint64_t>& seeds, double rmsd_tol);
}  // namespace b200

}  // namespace mdreduce
