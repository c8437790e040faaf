// dropin.cpp — the reference's C++ operator API (namespace mdreduce) over the
// B200 C-ABI.  Validation and exceptions follow the reference (thrown before
// any work); numerics run on the GPU through mdr.h.  Pure host logic of the
// API surface (Genotype accessors, BlockConfig, RngStream, MDRI parsing)
// is restated here from the reference's documented behaviour.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numbers>
#include <sstream>

#include "mdr.h"
#include "mdreduce_b200.hpp"

namespace mdreduce {
namespace {

struct Ctx {
  mdr_ctx* c = nullptr;
  int device = 0;
  ~Ctx() {
    if (c) mdr_ctx_destroy(c);
  }
};

thread_local int t_device = 0;
thread_local int t_pair = MDR_PAIR_FP64_FAST;
thread_local int t_exact = 0;

mdr_ctx* ctx() {
  thread_local std::unique_ptr<Ctx> holder;
  if (!holder || holder->device != t_device) {
    holder = std::make_unique<Ctx>();
    holder->device = t_device;
    holder->c = mdr_ctx_create(t_device);
    if (!holder->c) throw DeviceError("mdr_ctx_create failed: no usable CUDA device " + std::to_string(t_device));
  }
  mdr_ctx_set_pair_precision(holder->c, t_pair);
  mdr_ctx_set_exact_torsion(holder->c, t_exact);
  return holder->c;
}

void check(int rc) {
  if (rc == MDR_OK) return;
  const std::string msg = mdr_last_error(ctx());
  switch (rc) {
    case MDR_ERR_SIZE: throw SizeError(msg);
    case MDR_ERR_BLOCK_SIZE: throw UnsupportedBlockSizeError(msg);
    case MDR_ERR_NUMERIC_DOMAIN: throw NumericDomainError(msg);
    case MDR_ERR_PARSE: throw ParseError(0, msg);
    case MDR_ERR_CUDA: throw DeviceError(msg);
    default: throw std::invalid_argument(msg);
  }
}

int method_id(ReduceMethod m) {
  return m == ReduceMethod::Baseline ? MDR_METHOD_BASELINE : m == ReduceMethod::Tcu ? MDR_METHOD_TCU : MDR_METHOD_TCU_SPLIT;
}
int accum_id(AccumMode a) { return a == AccumMode::Half ? MDR_ACCUM_HALF : MDR_ACCUM_SINGLE; }

SyncStats to_stats(const mdr_sync_stats& s) {
  SyncStats o;
  o.block_syncs = s.block_syncs;
  o.warp_shuffles = s.warp_shuffles;
  o.atomic_adds = s.atomic_adds;
  o.memory_fences = s.memory_fences;
  o.mma_ops = s.mma_ops;
  o.shared_mem_bytes = s.shared_mem_bytes;
  o.precision_conversions = s.precision_conversions;
  return o;
}

// Flattened instance kept alive for the duration of a call.
struct FlatInstance {
  std::vector<double> atoms, sites;
  std::vector<int32_t> tors;
  mdr_instance c{};
  explicit FlatInstance(const LigandInstance& in) {
    for (const Atom& a : in.atoms) {
      atoms.insert(atoms.end(), {a.pos[0], a.pos[1], a.pos[2], a.weight});
      tors.push_back(a.torsion);
    }
    for (const Site& s : in.sites) sites.insert(sites.end(), {s.pos[0], s.pos[1], s.pos[2], s.depth, s.preferred_distance});
    c.n_atoms = static_cast<int32_t>(in.atoms.size());
    c.n_sites = static_cast<int32_t>(in.sites.size());
    c.n_rot = in.n_rot;
    c.atom_xyzw = atoms.data();
    c.atom_torsion = tors.data();
    c.site_xyzdd = sites.data();
  }
};

void check_genotype(const LigandInstance& in, const Genotype& g, const char* where) {  // docking.cpp:138-144
  if (static_cast<int>(g.torsions.size()) != in.n_rot)
    throw SizeError(std::string(where) + ": genotype has " + std::to_string(g.torsions.size()) +
                    " torsions, instance needs " + std::to_string(in.n_rot));
}

std::vector<double> flat_genotypes(const std::vector<Genotype>& gs) {
  std::vector<double> out;
  for (const Genotype& g : gs)
    for (int d = 0; d < g.dim(); ++d) out.push_back(g.get(d));
  return out;
}

Genotype make_genotype(const double* v, int n_rot) {
  Genotype g;
  g.torsions.resize(static_cast<std::size_t>(n_rot));
  for (int d = 0; d < 6 + n_rot; ++d) g.set(d, v[d]);
  return g;
}

double wrap_angle(double a) {  // docking.cpp:62-64
  return a - 2.0 * std::numbers::pi * std::floor((a + std::numbers::pi) / (2.0 * std::numbers::pi));
}

mdr_lga_settings to_c(const LgaSettings& s) {
  mdr_lga_settings o;
  o.population_size = s.population_size;
  o.generations = s.generations;
  o.max_evaluations = s.max_evaluations;
  o.ls_fraction = s.ls_fraction;
  o.ls_max_iters = s.ls_max_iters;
  o.partition = s.partition;
  o.ls_convergence_tol = s.ls_convergence_tol;
  o.mutation_sigma = s.mutation_sigma;
  return o;
}

}  // namespace

// ---------------------------------------------------------------- half / mma
Half f32_to_half(float v) {
  uint16_t h = 0;
  check(mdr_f32_to_half_batch(ctx(), &v, 1, &h));
  return Half::from_bits(h);
}

float half_to_f32(Half h) {
  const uint16_t b = h.bits();
  float f = 0.0f;
  check(mdr_half_to_f32_batch(ctx(), &b, 1, &f));
  return f;
}

Half half_add(Half a, Half b) { return f32_to_half(half_to_f32(a) + half_to_f32(b)); }

Mat16 load_matrix(std::span<const Half> src, Layout layout) {  // mma.cpp:10-26
  if (src.size() != Mat16::kElems) throw SizeError("load_matrix expects 256 elements, got " + std::to_string(src.size()));
  Mat16 m;
  m.set_layout(layout);
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) m.set(i, j, src[layout == Layout::RowMajor ? i * 16 + j : j * 16 + i]);
  return m;
}

std::vector<float> store_matrix(const Accum16& acc, Layout layout) {  // mma.cpp:28-39
  std::vector<float> out(Mat16::kElems);
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) out[layout == Layout::RowMajor ? i * 16 + j : j * 16 + i] = acc.at(i, j);
  return out;
}

Accum16 mma(const Mat16& a, const Mat16& b, const Accum16& c) {
  uint16_t ab[256], bb[256];
  for (int i = 0; i < 256; ++i) {
    ab[i] = a.data()[i].bits();
    bb[i] = b.data()[i].bits();
  }
  Accum16 d(c.mode());
  float out[256];
  check(mdr_mma_batch(ctx(), ab, bb, c.data(), 1, accum_id(c.mode()), out));
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) d.set(i, j, out[i * 16 + j]);
  return d;
}

// ---------------------------------------------------------------- reduce
Mat16 make_p() {  // reduce.cpp:12-21
  Mat16 p;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) p.set(i, j, Half::from_bits(0x3C00));
  return p;
}

Mat16 make_q() {  // reduce.cpp:23-34
  Mat16 q;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j)
      if ((i & 3) == (j & 3)) q.set(i, j, Half::from_bits(0x3C00));
  return q;
}

Mat16 pack_vectors(std::span<const Vec4> vs) {  // reduce.cpp:36-51
  if (vs.empty() || vs.size() > 64) throw SizeError("pack_vectors expects 1 to 64 vectors, got " + std::to_string(vs.size()));
  std::vector<float> f(4 * vs.size());
  for (std::size_t j = 0; j < vs.size(); ++j) {
    f[4 * j] = vs[j].x;
    f[4 * j + 1] = vs[j].y;
    f[4 * j + 2] = vs[j].z;
    f[4 * j + 3] = vs[j].e;
  }
  std::vector<uint16_t> h(f.size());
  check(mdr_f32_to_half_batch(ctx(), f.data(), f.size(), h.data()));
  std::vector<Half> flat(Mat16::kElems);
  for (std::size_t i = 0; i < h.size(); ++i) flat[i] = Half::from_bits(h[i]);
  return load_matrix(flat, Layout::ColMajor);
}

std::pair<Vec4, SyncStats> reduce4(std::span<const Vec4> vs, AccumMode mode) {
  if (vs.empty()) throw SizeError("reduce4 requires at least one vector");
  float out[4];
  mdr_sync_stats st;
  check(mdr_reduce4_batch(ctx(), reinterpret_cast<const float*>(vs.data()), static_cast<int>(vs.size()), 1,
                          MDR_METHOD_TCU, accum_id(mode), out, &st));
  return {Vec4{out[0], out[1], out[2], out[3]}, to_stats(st)};
}

std::pair<float, SyncStats> baseline_warp_reduce(std::span<const float> lanes) {
  if (lanes.size() != 32) throw SizeError("baseline_warp_reduce expects exactly 32 lanes, got " + std::to_string(lanes.size()));
  float out;
  mdr_sync_stats st;
  check(mdr_warp_reduce_batch(ctx(), lanes.data(), 1, &out, &st));
  return {out, to_stats(st)};
}

std::pair<float, SyncStats> baseline_block_reduce(std::span<const float> values, int threads) {
  float out = 0.0f;
  mdr_sync_stats st;
  check(mdr_block_reduce_batch(ctx(), values.data(), threads, 0, &out, &st));  // block-size validation first
  if (values.size() != static_cast<std::size_t>(threads))
    throw SizeError("baseline_block_reduce got " + std::to_string(values.size()) + " values for " +
                    std::to_string(threads) + " threads");
  check(mdr_block_reduce_batch(ctx(), values.data(), threads, 1, &out, &st));
  return {out, to_stats(st)};
}

std::pair<std::array<float, 7>, SyncStats> reduce7(std::span<const Partial7> records, ReduceMethod method,
                                                   AccumMode accum_mode) {
  std::array<float, 7> out{};
  mdr_sync_stats st;
  check(mdr_reduce7_batch(ctx(), reinterpret_cast<const float*>(records.data()), static_cast<int>(records.size()), 1,
                          method_id(method), accum_id(accum_mode), out.data(), &st));
  return {out, to_stats(st)};
}

BlockConfig::BlockConfig(int threads, ReduceMethod m, AccumMode a)  // simblock.cpp:10-19
    : threads_per_block(threads), method(m), accum_mode(a) {
  const int lo = m == ReduceMethod::Tcu ? 64 : 32;
  if (threads < lo || threads > 1024 || threads % 32 != 0)
    throw UnsupportedBlockSizeError(std::string(m == ReduceMethod::Tcu ? "tcu" : "baseline") +
                                    " blocks support multiples of 32 in [" + std::to_string(lo) + ", 1024], got " +
                                    std::to_string(threads));
}

// One block through the configured method (simblock.cpp:21-58): Tcu ->
// reduce4; Baseline -> one baseline block reduction per component (a single
// device launch of mdr_reduce4_batch with method BASELINE).
std::pair<Vec4, SyncStats> simulate_block(const BlockConfig& cfg, std::span<const Vec4> values) {
  if (values.size() != static_cast<std::size_t>(cfg.threads_per_block))
    throw SizeError("simulate_block got " + std::to_string(values.size()) + " records for " +
                    std::to_string(cfg.threads_per_block) + " threads");
  if (cfg.method == ReduceMethod::Tcu) return reduce4(values, cfg.accum_mode);
  float out[4];
  mdr_sync_stats st;
  check(mdr_reduce4_batch(ctx(), reinterpret_cast<const float*>(values.data()), static_cast<int>(values.size()), 1,
                          method_id(cfg.method), accum_id(cfg.accum_mode), out, &st));
  return {Vec4{out[0], out[1], out[2], out[3]}, to_stats(st)};
}

std::pair<std::array<float, 7>, SyncStats> simulate_block(const BlockConfig& cfg, std::span<const Partial7> values) {
  if (values.size() != static_cast<std::size_t>(cfg.threads_per_block))
    throw SizeError("simulate_block got " + std::to_string(values.size()) + " records for " +
                    std::to_string(cfg.threads_per_block) + " threads");
  return reduce7(values, cfg.method, cfg.accum_mode);
}

double estimate_cost(const SyncStats& st, const CostWeights& w) {  // simblock.cpp:60-66
  return static_cast<double>(st.block_syncs) * w.block_sync + static_cast<double>(st.atomic_adds) * w.atomic +
         static_cast<double>(st.warp_shuffles) * w.shuffle + static_cast<double>(st.memory_fences) * w.fence +
         static_cast<double>(st.mma_ops) * w.mma;
}

// Counter profile of one baseline block reduction vs one tcu reduce4 per
// block size (simblock.cpp:68-98), both obtained from the device calls.
std::vector<SweepRow> scaling_sweep(std::span<const int> sizes, const CostWeights& w, AccumMode accum) {
  std::vector<SweepRow> rows;
  for (const int n : sizes) {
    const BlockConfig tcu_cfg(n, ReduceMethod::Tcu, accum), base_cfg(n, ReduceMethod::Baseline, accum);
    (void)tcu_cfg;
    (void)base_cfg;
    SweepRow row;
    row.threads_per_block = n;
    row.baseline = baseline_block_reduce(std::vector<float>(static_cast<std::size_t>(n), 0.0f), n).second;
    row.tcu = reduce4(std::vector<Vec4>(static_cast<std::size_t>(n)), accum).second;
    row.cost_baseline = estimate_cost(row.baseline, w);
    row.cost_tcu = estimate_cost(row.tcu, w);
    row.degenerate = row.cost_tcu == 0.0;
    row.cost_ratio = row.degenerate ? 1.0 : row.cost_baseline / row.cost_tcu;
    rows.push_back(row);
  }
  return rows;
}

// ---------------------------------------------------------------- rng
namespace {
std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
std::uint64_t fnv1a(std::string_view s) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (unsigned char c : s) h = (h ^ c) * 0x100000001b3ull;
  return h;
}
}  // namespace

RngStream::RngStream(std::uint64_t seed, std::string_view label) : key_(mix64(seed ^ mix64(fnv1a(label)))) {}
std::uint64_t RngStream::next_u64() { return mix64(key_ + (++counter_) * 0x9e3779b97f4a7c15ull); }
double RngStream::next_double() { return static_cast<double>(next_u64() >> 11) * 0x1p-53; }
double RngStream::uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
double RngStream::normal() {
  const double u1 = static_cast<double>((next_u64() >> 11) + 1) * 0x1p-53;
  const double u2 = next_double();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
}
std::uint64_t RngStream::next_index(std::uint64_t n) { return n == 0 ? 0 : next_u64() % n; }

// ---------------------------------------------------------------- MDRI I/O
LigandInstance parse_instance(std::string_view text) {  // instance_io.cpp:137-253 (behaviour)
  LigandInstance inst;
  bool magic = false, saw_nrot = false;
  std::vector<int> atom_lines;
  int line_no = 0;
  std::size_t pos = 0;
  auto number = [](const std::string& t, int ln, const char* what) {
    char* end = nullptr;
    const double v = std::strtod(t.c_str(), &end);
    if (t.empty() || *end != '\0') throw ParseError(ln, std::string("invalid number for ") + what + ": '" + t + "'");
    if (!std::isfinite(v)) throw ParseError(ln, std::string("non-finite value for ") + what);
    return v;
  };
  auto integer = [](const std::string& t, int ln, const char* what) {
    char* end = nullptr;
    const long v = std::strtol(t.c_str(), &end, 10);
    if (t.empty() || *end != '\0') throw ParseError(ln, std::string("invalid integer for ") + what + ": '" + t + "'");
    return v;
  };
  while (pos <= text.size()) {
    const std::size_t eol = text.find('\n', pos);
    std::string line(text.substr(pos, eol == std::string_view::npos ? text.size() - pos : eol - pos));
    pos = eol == std::string_view::npos ? text.size() + 1 : eol + 1;
    ++line_no;
    if (const auto h = line.find('#'); h != std::string::npos) line.resize(h);
    std::istringstream ss(line);
    std::vector<std::string> tok;
    for (std::string t; ss >> t;) tok.push_back(t);
    if (!magic) {
      if (tok.empty()) {
        if (line_no == 1) throw ParseError(1, "missing magic line 'MDRI 1'");
        continue;
      }
      if (tok.size() != 2 || tok[0] != "MDRI" || tok[1] != "1") throw ParseError(line_no, "missing magic line 'MDRI 1'");
      magic = true;
      continue;
    }
    if (tok.empty()) continue;
    if (tok[0] == "nrot") {
      if (saw_nrot) throw ParseError(line_no, "duplicate nrot line");
      if (tok.size() != 2) throw ParseError(line_no, "nrot expects one integer");
      const long n = integer(tok[1], line_no, "nrot");
      if (n < 0) throw ParseError(line_no, "nrot must be non-negative");
      inst.n_rot = static_cast<int>(n);
      saw_nrot = true;
    } else if (tok[0] == "atom") {
      if (tok.size() != 6) throw ParseError(line_no, "atom expects <x> <y> <z> <weight> <torsion|->");
      Atom a;
      for (int k = 0; k < 3; ++k) a.pos[k] = number(tok[1 + k], line_no, "atom coordinate");
      a.weight = number(tok[4], line_no, "atom weight");
      if (a.weight <= 0.0) throw ParseError(line_no, "atom weight must be positive");
      if (tok[5] == "-") {
        a.torsion = -1;
      } else {
        const long t = integer(tok[5], line_no, "torsion index");
        if (t < 0) throw ParseError(line_no, "torsion index must be non-negative or '-'");
        a.torsion = static_cast<int>(t);
      }
      inst.atoms.push_back(a);
      atom_lines.push_back(line_no);
    } else if (tok[0] == "site") {
      if (tok.size() != 6) throw ParseError(line_no, "site expects <x> <y> <z> <depth> <d0>");
      Site s;
      for (int k = 0; k < 3; ++k) s.pos[k] = number(tok[1 + k], line_no, "site coordinate");
      s.depth = number(tok[4], line_no, "site depth");
      s.preferred_distance = number(tok[5], line_no, "site d0");
      if (s.depth <= 0.0) throw ParseError(line_no, "site depth must be positive");
      if (s.preferred_distance <= 0.0) throw ParseError(line_no, "site d0 must be positive");
      inst.sites.push_back(s);
    } else {
      throw ParseError(line_no, "unknown directive '" + tok[0] + "'");
    }
  }
  if (!magic) throw ParseError(1, "missing magic line 'MDRI 1'");
  if (!saw_nrot) throw ParseError(line_no, "missing nrot line");
  for (std::size_t i = 0; i < inst.atoms.size(); ++i)
    if (inst.atoms[i].torsion >= inst.n_rot)
      throw ParseError(atom_lines[i], "atom references torsion " + std::to_string(inst.atoms[i].torsion) +
                                          " but nrot is " + std::to_string(inst.n_rot));
  if (inst.atoms.empty()) throw ParseError(line_no, "instance needs at least one atom");
  if (inst.sites.empty()) throw ParseError(line_no, "instance needs at least one site");
  return inst;
}

std::string serialize_instance(const LigandInstance& in) {
  std::ostringstream o;
  o.precision(17);
  o << "MDRI 1\nnrot " << in.n_rot << "\n";
  for (const Atom& a : in.atoms) {
    o << "atom " << a.pos[0] << ' ' << a.pos[1] << ' ' << a.pos[2] << ' ' << a.weight << ' ';
    if (a.torsion < 0)
      o << '-';
    else
      o << a.torsion;
    o << '\n';
  }
  for (const Site& s : in.sites)
    o << "site " << s.pos[0] << ' ' << s.pos[1] << ' ' << s.pos[2] << ' ' << s.depth << ' ' << s.preferred_distance
      << '\n';
  return o.str();
}

// ---------------------------------------------------------------- results CSV
namespace {
constexpr std::string_view kResultHeader =
    "seed,method,accum_mode,instance,best_energy,evaluations,converged,block_syncs,atomic_adds,mma_ops";

std::string csv_text(std::string_view s) {  // quoted only when needed, "" escapes
  if (s.find_first_of(",\"\n") == std::string_view::npos) return std::string(s);
  std::string q = "\"";
  for (const char c : s) q += c == '"' ? std::string("\"\"") : std::string(1, c);
  return q + "\"";
}

std::string num17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

template <class T>
T parse_num(const std::string& f, int line, const char* what) {
  T v{};
  const auto [p, ec] = std::from_chars(f.data(), f.data() + f.size(), v);
  if (ec != std::errc() || p != f.data() + f.size())
    throw ParseError(line, std::string("bad ") + what + " '" + f + "'");
  return v;
}
}  // namespace

std::string write_results(std::span<const ResultRow> rows) {
  std::string out(kResultHeader);
  out += '\n';
  for (const ResultRow& r : rows)
    out += std::to_string(r.seed) + ',' + csv_text(r.method) + ',' + csv_text(r.accum_mode) + ',' +
           csv_text(r.instance) + ',' + num17(r.best_energy) + ',' + std::to_string(r.evaluations) + ',' +
           (r.converged ? "true" : "false") + ',' + std::to_string(r.block_syncs) + ',' +
           std::to_string(r.atomic_adds) + ',' + std::to_string(r.mma_ops) + '\n';
  return out;
}

std::vector<ResultRow> parse_results(std::string_view csv) {
  std::vector<ResultRow> rows;
  bool header = false;
  int line = 0;
  std::size_t pos = 0;
  while (pos < csv.size()) {
    // one record: up to the first newline outside quotes (quoted fields may
    // span lines; errors name the record's first line)
    const int first = ++line;
    std::vector<std::string> f(1);
    bool quoted = false, any = false;
    for (; pos < csv.size(); ++pos) {
      const char c = csv[pos];
      if (quoted) {
        if (c == '"') {
          if (pos + 1 < csv.size() && csv[pos + 1] == '"') {
            f.back() += '"';
            ++pos;
          } else {
            quoted = false;
          }
        } else {
          if (c == '\n') ++line;
          f.back() += c;
        }
      } else if (c == '"') {
        if (!f.back().empty()) throw ParseError(first, "unexpected quote inside unquoted field");
        quoted = any = true;
      } else if (c == ',') {
        f.emplace_back();
        any = true;
      } else if (c == '\n') {
        ++pos;
        break;
      } else {
        f.back() += c;
        any = true;
      }
    }
    if (quoted) throw ParseError(first, "unterminated quoted field");
    if (!any) continue;  // empty line
    if (!header) {
      std::string joined;
      for (std::size_t i = 0; i < f.size(); ++i) joined += (i ? "," : "") + f[i];
      if (joined != kResultHeader) throw ParseError(first, "unexpected results header");
      header = true;
      continue;
    }
    if (f.size() != 10) throw ParseError(first, "expected 10 fields, got " + std::to_string(f.size()));
    ResultRow r;
    r.seed = parse_num<std::uint64_t>(f[0], first, "seed");
    r.method = f[1];
    r.accum_mode = f[2];
    r.instance = f[3];
    r.best_energy = parse_num<double>(f[4], first, "best_energy");
    r.evaluations = parse_num<std::int64_t>(f[5], first, "evaluations");
    if (f[6] != "true" && f[6] != "false") throw ParseError(first, "bad converged flag '" + f[6] + "'");
    r.converged = f[6] == "true";
    r.block_syncs = parse_num<std::uint64_t>(f[7], first, "block_syncs");
    r.atomic_adds = parse_num<std::uint64_t>(f[8], first, "atomic_adds");
    r.mma_ops = parse_num<std::uint64_t>(f[9], first, "mma_ops");
    rows.push_back(std::move(r));
  }
  if (!header) throw ParseError(1, "missing results header");
  return rows;
}

// ---------------------------------------------------------------- docking
double Genotype::get(int i) const {  // docking.cpp:148-158
  switch (i) {
    case 0: return x;
    case 1: return y;
    case 2: return z;
    case 3: return phi;
    case 4: return theta;
    case 5: return alpha;
    default: return torsions[static_cast<std::size_t>(i - 6)];
  }
}

void Genotype::set(int i, double v) {
  switch (i) {
    case 0: x = v; return;
    case 1: y = v; return;
    case 2: z = v; return;
    case 3: phi = v; return;
    case 4: theta = v; return;
    case 5: alpha = v; return;
    default: torsions[static_cast<std::size_t>(i - 6)] = v; return;
  }
}

void Genotype::normalize_angles() {
  phi = wrap_angle(phi);
  theta = wrap_angle(theta);
  alpha = wrap_angle(alpha);
  for (double& t : torsions) t = wrap_angle(t);
}

std::array<double, 3> torsion_axis(int k) {  // docking.cpp:181-189
  const double az = 2.399963229728653 * k + 0.3;
  const double zc = 0.5 + 0.35 * std::sin(0.9 * k + 0.4);
  const double v[3] = {0.8 * std::cos(az), 0.8 * std::sin(az), zc};
  const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  return {v[0] / n, v[1] / n, v[2] / n};
}

namespace b200 {

void set_device(int device) { t_device = device; }
void set_pair_mode(PairMode m) {
  t_pair = m == PairMode::Reference ? MDR_PAIR_FP64 : m == PairMode::Fp32 ? MDR_PAIR_FP32 : MDR_PAIR_FP64_FAST;
}

void set_exact_torsion(bool on) { t_exact = on ? 1 : 0; }

std::vector<ScoreResult> score_batch(const LigandInstance& in, const std::vector<Genotype>& poses, ReduceMethod method,
                                     AccumMode accum, int partition) {
  for (const Genotype& g : poses) check_genotype(in, g, "score");
  const BlockConfig cfg(partition, method == ReduceMethod::TcuSplit ? ReduceMethod::Baseline : method, accum);
  (void)cfg;
  FlatInstance fi(in);
  const int n = static_cast<int>(poses.size()), dim = 6 + in.n_rot;
  const std::vector<double> g = flat_genotypes(poses);
  std::vector<float> e(n), grad(static_cast<std::size_t>(n) * dim), tq(3 * static_cast<std::size_t>(n));
  mdr_sync_stats st;
  check(mdr_score_batch(ctx(), &fi.c, g.data(), n, method_id(method), accum_id(accum), partition, e.data(),
                        grad.data(), tq.data(), &st));
  std::vector<ScoreResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    ScoreResult& r = out[static_cast<std::size_t>(i)];
    r.energy = e[i];
    r.gradient.assign(grad.begin() + static_cast<std::ptrdiff_t>(i) * dim,
                      grad.begin() + static_cast<std::ptrdiff_t>(i + 1) * dim);
    r.torque = {tq[3 * i], tq[3 * i + 1], tq[3 * i + 2]};
    r.reduce_stats = to_stats(st);
  }
  return out;
}

std::vector<LocalSearchResult> local_search_batch(const LigandInstance& in, const std::vector<Genotype>& starts,
                                                  int max_iters, double tol, ReduceMethod method, AccumMode accum,
                                                  int partition) {
  for (const Genotype& g : starts) check_genotype(in, g, "score");
  FlatInstance fi(in);
  const int n = static_cast<int>(starts.size()), dim = 6 + in.n_rot;
  const std::vector<double> s = flat_genotypes(starts);
  std::vector<double> og(s.size()), oe(static_cast<std::size_t>(n));
  std::vector<int32_t> it(static_cast<std::size_t>(n)), cv(static_cast<std::size_t>(n));
  std::vector<mdr_sync_stats> st(static_cast<std::size_t>(std::max(n, 1)));
  check(mdr_local_search_batch(ctx(), &fi.c, s.data(), n, max_iters, tol, method_id(method), accum_id(accum), partition,
                               og.data(), oe.data(), it.data(), cv.data(), st.data()));
  std::vector<LocalSearchResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    LocalSearchResult& r = out[static_cast<std::size_t>(i)];
    r.genotype = make_genotype(og.data() + static_cast<std::ptrdiff_t>(i) * dim, in.n_rot);
    r.energy = oe[i];
    r.iterations = it[i];
    r.converged = cv[i] != 0;
    r.stats = to_stats(st[i]);
  }
  return out;
}

std::vector<DockResult> lga_run_batch(const LigandInstance& in, ReduceMethod method, AccumMode accum,
                                      const LgaSettings& settings, const std::vector<std::uint64_t>& seeds) {
  FlatInstance fi(in);
  const mdr_lga_settings cs = to_c(settings);
  const int n = static_cast<int>(seeds.size()), dim = 6 + in.n_rot;
  if (settings.population_size < 2) throw SizeError("lga_run needs a population of at least 2");
  const int maxr = mdr_lga_max_records(&cs);
  std::vector<double> be(static_cast<std::size_t>(n)), bg(static_cast<std::size_t>(n) * dim);
  std::vector<int64_t> ev(static_cast<std::size_t>(n));
  std::vector<int32_t> cv(static_cast<std::size_t>(n)), nr(static_cast<std::size_t>(n));
  std::vector<mdr_ls_record> recs(static_cast<std::size_t>(n) * maxr);
  std::vector<mdr_sync_stats> st(static_cast<std::size_t>(std::max(n, 1)));
  check(mdr_lga_run_batch(ctx(), &fi.c, method_id(method), accum_id(accum), &cs, seeds.data(), n, be.data(), bg.data(),
                          ev.data(), cv.data(), nr.data(), recs.data(), st.data()));
  std::vector<DockResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    DockResult& r = out[static_cast<std::size_t>(i)];
    r.best_energy = be[i];
    r.best_genotype = make_genotype(bg.data() + static_cast<std::ptrdiff_t>(i) * dim, in.n_rot);
    r.evaluations = ev[i];
    r.converged = cv[i] != 0;
    for (int k = 0; k < std::min<int>(nr[i], maxr); ++k) {
      const mdr_ls_record& q = recs[static_cast<std::size_t>(i) * maxr + k];
      r.runs.push_back(LsRunRecord{q.best_energy, q.iterations, q.converged != 0});
    }
    r.total_stats = to_stats(st[i]);
  }
  return out;
}

// ---------------------------------------------------------------- grid mode
namespace {
mdr_grid grid_to_c(const GridShape& g, const float* maps) {
  mdr_grid o{};
  o.nx = g.nx;
  o.ny = g.ny;
  o.nz = g.nz;
  o.n_types = g.n_types;
  o.origin[0] = g.origin[0];
  o.origin[1] = g.origin[1];
  o.origin[2] = g.origin[2];
  o.spacing = g.spacing;
  o.maps = maps;
  return o;
}

struct FlatChem {  // mdr_ligand_params view of a LigandChemistry
  mdr_ligand_params c{};
  explicit FlatChem(const LigandInstance& in, const LigandChemistry& ch) {
    const std::size_t n = in.atoms.size();
    if (ch.atom_type.size() != n || ch.charge.size() != n || ch.radius.size() != n || ch.epsilon.size() != n)
      throw SizeError("ligand chemistry needs one entry per atom");
    c.atom_type = reinterpret_cast<const int32_t*>(ch.atom_type.data());
    c.atom_charge = ch.charge.data();
    c.atom_radius = ch.radius.data();
    c.atom_epsilon = ch.epsilon.data();
    c.elec_scale = ch.elec_scale;
    c.intra = ch.intra ? 1 : 0;
  }
};

std::shared_ptr<void> grid_handle(mdr_dev_grid* h) {
  if (!h) check(MDR_ERR_CUDA);
  return std::shared_ptr<void>(h, [](void* p) { mdr_grid_free(nullptr, static_cast<mdr_dev_grid*>(p)); });
}

mdr_dev_grid* dev_grid(const Receptor& r) { return static_cast<mdr_dev_grid*>(r.handle()); }
}  // namespace

Receptor Receptor::upload(const GridMaps& m) {
  const std::size_t need = static_cast<std::size_t>(m.shape.n_types + 2) * m.shape.nx * m.shape.ny * m.shape.nz;
  if (m.maps.size() != need) throw SizeError("grid maps need (n_types + 2) * nx * ny * nz values");
  const mdr_grid g = grid_to_c(m.shape, m.maps.data());
  Receptor r;
  r.shape_ = m.shape;
  mdr_dev_grid* h = mdr_grid_upload(ctx(), &g);
  if (!h) check(MDR_ERR_SIZE);
  r.handle_ = grid_handle(h);
  return r;
}

Receptor Receptor::build(const LigandInstance& sites, const ReceptorFields& f, const GridShape& shape) {
  if (f.site_charge.size() != sites.sites.size() || f.site_volume.size() != sites.sites.size() ||
      static_cast<int>(f.type_depth_scale.size()) != shape.n_types ||
      static_cast<int>(f.type_dist_scale.size()) != shape.n_types)
    throw SizeError("receptor fields need one entry per site / type");
  FlatInstance fi(sites);
  mdr_receptor_fields c{f.site_charge.data(), f.site_volume.data(), f.type_depth_scale.data(),
                        f.type_dist_scale.data(), f.elec_scale, f.desolv_sigma};
  const mdr_grid g = grid_to_c(shape, nullptr);
  Receptor r;
  r.shape_ = shape;
  mdr_dev_grid* h = mdr_grid_build(ctx(), &fi.c, &c, &g);
  if (!h) check(MDR_ERR_SIZE);
  r.handle_ = grid_handle(h);
  return r;
}

GridMaps Receptor::download() const {
  GridMaps m;
  m.shape = shape_;
  m.maps.resize(static_cast<std::size_t>(shape_.n_types + 2) * shape_.nx * shape_.ny * shape_.nz);
  check(mdr_grid_download(ctx(), dev_grid(*this), m.maps.data()));
  return m;
}

std::vector<ScoreResult> grid_score_batch(const Receptor& rec, const LigandInstance& in, const LigandChemistry& ch,
                                          const std::vector<Genotype>& poses, ReduceMethod method, int partition) {
  for (const Genotype& g : poses) check_genotype(in, g, "score");
  FlatInstance fi(in);
  FlatChem fc(in, ch);
  const int n = static_cast<int>(poses.size()), dim = 6 + in.n_rot;
  const std::vector<double> g = flat_genotypes(poses);
  std::vector<float> e(n), grad(static_cast<std::size_t>(n) * dim), tq(3 * static_cast<std::size_t>(n));
  check(mdr_grid_score_batch(ctx(), dev_grid(rec), &fi.c, &fc.c, g.data(), n, method_id(method), partition, e.data(),
                             grad.data(), tq.data()));
  std::vector<ScoreResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    ScoreResult& r = out[static_cast<std::size_t>(i)];
    r.energy = e[i];
    r.gradient.assign(grad.begin() + static_cast<std::ptrdiff_t>(i) * dim,
                      grad.begin() + static_cast<std::ptrdiff_t>(i + 1) * dim);
    r.torque = {tq[3 * i], tq[3 * i + 1], tq[3 * i + 2]};
  }
  return out;
}

std::vector<LocalSearchResult> grid_local_search_batch(const Receptor& rec, const LigandInstance& in,
                                                       const LigandChemistry& ch, const std::vector<Genotype>& starts,
                                                       int max_iters, double tol, ReduceMethod method, int partition) {
  for (const Genotype& g : starts) check_genotype(in, g, "score");
  FlatInstance fi(in);
  FlatChem fc(in, ch);
  const int n = static_cast<int>(starts.size()), dim = 6 + in.n_rot;
  const std::vector<double> s = flat_genotypes(starts);
  std::vector<double> og(s.size()), oe(static_cast<std::size_t>(n));
  std::vector<int32_t> it(static_cast<std::size_t>(n)), cv(static_cast<std::size_t>(n));
  check(mdr_grid_local_search_batch(ctx(), dev_grid(rec), &fi.c, &fc.c, s.data(), n, max_iters, tol,
                                    method_id(method), partition, og.data(), oe.data(), it.data(), cv.data()));
  std::vector<LocalSearchResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    LocalSearchResult& r = out[static_cast<std::size_t>(i)];
    r.genotype = make_genotype(og.data() + static_cast<std::ptrdiff_t>(i) * dim, in.n_rot);
    r.energy = oe[i];
    r.iterations = it[i];
    r.converged = cv[i] != 0;
  }
  return out;
}

std::vector<DockResult> grid_lga_run_batch(const Receptor& rec, const LigandInstance& in, const LigandChemistry& ch,
                                           ReduceMethod method, const LgaSettings& settings,
                                           const std::vector<std::uint64_t>& seeds) {
  FlatInstance fi(in);
  FlatChem fc(in, ch);
  const mdr_lga_settings cs = to_c(settings);
  if (settings.population_size < 2) throw SizeError("lga_run needs a population of at least 2");
  const int n = static_cast<int>(seeds.size()), dim = 6 + in.n_rot, maxr = mdr_lga_max_records(&cs);
  std::vector<double> be(static_cast<std::size_t>(n)), bg(static_cast<std::size_t>(n) * dim);
  std::vector<int64_t> ev(static_cast<std::size_t>(n));
  std::vector<int32_t> cv(static_cast<std::size_t>(n)), nr(static_cast<std::size_t>(n));
  std::vector<mdr_ls_record> recs(static_cast<std::size_t>(n) * maxr);
  check(mdr_grid_lga_run_batch(ctx(), dev_grid(rec), &fi.c, &fc.c, method_id(method), &cs, seeds.data(), n,
                               be.data(), bg.data(), ev.data(), cv.data(), nr.data(), recs.data()));
  std::vector<DockResult> out(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    DockResult& r = out[static_cast<std::size_t>(i)];
    r.best_energy = be[i];
    r.best_genotype = make_genotype(bg.data() + static_cast<std::ptrdiff_t>(i) * dim, in.n_rot);
    r.evaluations = ev[i];
    r.converged = cv[i] != 0;
    for (int k = 0; k < std::min<int>(nr[i], maxr); ++k) {
      const mdr_ls_record& q = recs[static_cast<std::size_t>(i) * maxr + k];
      r.runs.push_back(LsRunRecord{q.best_energy, q.iterations, q.converged != 0});
    }
  }
  return out;
}

// ---------------------------------------------------------------- clustering
std::vector<std::array<double, 3>> pose_coordinates(const LigandInstance& in, const Genotype& g) {
  check_genotype(in, g, "pose_coordinates");
  FlatInstance fi(in);
  const std::vector<double> gv = flat_genotypes({g});
  std::vector<double> xyz(3 * in.atoms.size());
  check(mdr_pose_coords_batch(ctx(), &fi.c, gv.data(), 1, xyz.data()));
  std::vector<std::array<double, 3>> out(in.atoms.size());
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return out;
}

Clustering cluster_poses(const LigandInstance& in, const std::vector<Genotype>& poses,
                         const std::vector<double>& energies, double tol) {
  if (energies.size() != poses.size()) throw SizeError("cluster_poses needs one energy per pose");
  for (const Genotype& g : poses) check_genotype(in, g, "cluster_poses");
  FlatInstance fi(in);
  const std::vector<double> gv = flat_genotypes(poses);
  Clustering c;
  c.cluster_of.resize(poses.size());
  c.rmsd_to_seed.resize(poses.size());
  int32_t nc = 0;
  check(mdr_cluster_poses(ctx(), &fi.c, gv.data(), energies.data(), static_cast<int>(poses.size()), tol,
                          reinterpret_cast<int32_t*>(c.cluster_of.data()), c.rmsd_to_seed.data(), &nc));
  c.n_clusters = nc;
  return c;
}

// ---------------------------------------------------------------- screen
std::vector<ScreenResult> screen_batch(const Receptor& rec, const std::vector<LigandInstance>& ligs,
                                       const std::vector<LigandChemistry>& chem, int runs, ReduceMethod method,
                                       const LgaSettings& settings, const std::vector<std::uint64_t>& seeds,
                                       double tol) {
  if (chem.size() != ligs.size()) throw SizeError("screen_batch needs chemistry per ligand");
  if (seeds.size() != ligs.size() * static_cast<std::size_t>(runs)) throw SizeError("one seed per (ligand, run)");
  std::vector<std::unique_ptr<FlatInstance>> fis;
  std::vector<std::unique_ptr<FlatChem>> fcs;
  std::vector<mdr_instance> ci;
  std::vector<mdr_ligand_params> cp;
  std::size_t gtot = 0;
  for (std::size_t j = 0; j < ligs.size(); ++j) {
    fis.push_back(std::make_unique<FlatInstance>(ligs[j]));
    fcs.push_back(std::make_unique<FlatChem>(ligs[j], chem[j]));
    ci.push_back(fis.back()->c);
    cp.push_back(fcs.back()->c);
    gtot += static_cast<std::size_t>(runs) * (6 + ligs[j].n_rot);
  }
  const std::size_t R = seeds.size();
  const mdr_lga_settings cs = to_c(settings);
  std::vector<double> be(R), bg(gtot), rm(R);
  std::vector<int64_t> ev(R);
  std::vector<int32_t> cv(R), cl(R), nc(ligs.size());
  check(mdr_grid_screen_batch(ctx(), dev_grid(rec), ci.data(), cp.data(), static_cast<int>(ligs.size()), runs,
                              method_id(method), &cs, seeds.data(), tol, be.data(), bg.data(), ev.data(), cv.data(),
                              cl.data(), rm.data(), nc.data()));
  std::vector<ScreenResult> out(ligs.size());
  std::size_t o = 0;
  for (std::size_t j = 0; j < ligs.size(); ++j) {
    ScreenResult& r = out[j];
    const int dim = 6 + ligs[j].n_rot;
    for (int k = 0; k < runs; ++k, o += static_cast<std::size_t>(dim)) {
      const std::size_t i = j * static_cast<std::size_t>(runs) + static_cast<std::size_t>(k);
      r.best_energy.push_back(be[i]);
      r.best_genotype.push_back(make_genotype(bg.data() + o, ligs[j].n_rot));
      r.evaluations.push_back(ev[i]);
      r.converged.push_back(cv[i] != 0);
      r.clusters.cluster_of.push_back(cl[i]);
      r.clusters.rmsd_to_seed.push_back(rm[i]);
    }
    r.clusters.n_clusters = nc[j];
  }
  return out;
}

}  // namespace b200

ScoreResult score(const LigandInstance& in, const Genotype& g, ReduceMethod method, AccumMode accum, int partition) {
  check_genotype(in, g, "score");
  return b200::score_batch(in, {g}, method, accum, partition)[0];
}

RefScore score_reference(const LigandInstance& in, const Genotype& g) {
  check_genotype(in, g, "score_reference");
  FlatInstance fi(in);
  const int dim = g.dim();
  std::vector<double> gv(static_cast<std::size_t>(dim)), grad(static_cast<std::size_t>(dim));
  for (int d = 0; d < dim; ++d) gv[d] = g.get(d);
  double e = 0.0, tq[3];
  check(mdr_score_reference_batch(ctx(), &fi.c, gv.data(), 1, &e, grad.data(), tq));
  RefScore r;
  r.energy = e;
  r.gradient = grad;
  r.torque = {tq[0], tq[1], tq[2]};
  return r;
}

AdadeltaState AdadeltaState::fresh(int dim, double rho, double epsilon) {
  AdadeltaState s;
  s.avg_sq_grad.assign(static_cast<std::size_t>(dim), 0.0);
  s.avg_sq_update.assign(static_cast<std::size_t>(dim), 0.0);
  s.rho = rho;
  s.epsilon = epsilon;
  return s;
}

std::pair<AdadeltaState, Genotype> adadelta_step(const AdadeltaState& state, const Genotype& g,
                                                 const std::vector<double>& grad) {
  const std::size_t dim = static_cast<std::size_t>(g.dim());
  if (grad.size() != dim || state.avg_sq_grad.size() != dim || state.avg_sq_update.size() != dim)
    throw SizeError("adadelta_step: state/gradient dimensions do not match genotype");
  AdadeltaState next = state;
  std::vector<double> gv(dim);
  for (std::size_t i = 0; i < dim; ++i) gv[i] = g.get(static_cast<int>(i));
  check(mdr_adadelta_step_batch(ctx(), static_cast<int>(dim), 1, state.rho, state.epsilon, next.avg_sq_grad.data(),
                                next.avg_sq_update.data(), gv.data(), grad.data()));
  return {next, make_genotype(gv.data(), static_cast<int>(g.torsions.size()))};
}

LocalSearchResult local_search(const LigandInstance& in, const Genotype& start, int max_iters, double tol,
                               ReduceMethod method, AccumMode accum, int partition, std::uint64_t /*rng_seed*/) {
  check_genotype(in, start, "score");
  return b200::local_search_batch(in, {start}, max_iters, tol, method, accum, partition)[0];
}

DockResult lga_run(const LigandInstance& in, ReduceMethod method, AccumMode accum, const LgaSettings& settings,
                   std::uint64_t seed) {
  return b200::lga_run_batch(in, method, accum, settings, {seed})[0];
}

namespace {
MethodSummary summarize(std::vector<double> b, int nonconv, int n) {  // docking.cpp:521-542
  std::sort(b.begin(), b.end());
  auto q = [&](double p) {
    if (b.size() == 1) return b[0];
    const double h = p * static_cast<double>(b.size() - 1);
    const std::size_t lo = static_cast<std::size_t>(h);
    const std::size_t hi = std::min(lo + 1, b.size() - 1);
    return b[lo] + (h - static_cast<double>(lo)) * (b[hi] - b[lo]);
  };
  MethodSummary s;
  s.min = b.front();
  s.q1 = q(0.25);
  s.median = q(0.5);
  s.q3 = q(0.75);
  s.max = b.back();
  double sum = 0.0;
  for (double x : b) sum += x;
  s.mean = sum / static_cast<double>(b.size());
  s.nonconvergent_fraction = static_cast<double>(nonconv) / static_cast<double>(n);
  return s;
}
}  // namespace

ValidationReport validate_pair(const LigandInstance& in, ReduceMethod ref_m, ReduceMethod test_m, AccumMode accum,
                               int n_runs, std::uint64_t base_seed, const LgaSettings& settings) {
  if (n_runs < 1) throw SizeError("validate_pair needs at least one run");
  std::vector<std::uint64_t> seeds(static_cast<std::size_t>(n_runs));
  for (int i = 0; i < n_runs; ++i) seeds[static_cast<std::size_t>(i)] = base_seed + static_cast<std::uint64_t>(i);
  const auto a = b200::lga_run_batch(in, ref_m, accum, settings, seeds);
  const auto b = b200::lga_run_batch(in, test_m, accum, settings, seeds);
  std::vector<double> ra, rb;
  int na = 0, nb = 0;
  for (int i = 0; i < n_runs; ++i) {
    ra.push_back(a[static_cast<std::size_t>(i)].best_energy);
    rb.push_back(b[static_cast<std::size_t>(i)].best_energy);
    na += a[static_cast<std::size_t>(i)].converged ? 0 : 1;
    nb += b[static_cast<std::size_t>(i)].converged ? 0 : 1;
  }
  ValidationReport rep;
  rep.n_runs = n_runs;
  rep.ref = summarize(ra, na, n_runs);
  rep.test = summarize(rb, nb, n_runs);
  rep.abs_diff_means = std::abs(rep.test.mean - rep.ref.mean);
  rep.relative_error =
      rep.ref.mean == 0.0 ? std::numeric_limits<double>::infinity() : rep.abs_diff_means / std::abs(rep.ref.mean);
  return rep;
}

}  // namespace mdreduce
