// test_dropin.cpp — the reference's C++ test scenarios (proj/tests/
// test_{half,mma,reduce,docking}.cpp, acceptance.cpp) written against the
// drop-in header mdreduce_b200.hpp and run on the GPU.  Same calls, same
// expected values; where hardware accumulation order legitimately differs
// (Tcu method) the tolerance is stated inline.
// Usage: test_dropin <dir with s1.mdri s2.mdri s3.mdri>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "mdreduce_b200.hpp"

using namespace mdreduce;

static int g_fail = 0, g_checks = 0;
static std::string g_data;

#define CHECK(cond)                                                         \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);         \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                            \
  do {                                                                      \
    ++g_checks;                                                             \
    bool _ok = false;                                                       \
    try {                                                                   \
      (void)(expr);                                                         \
    } catch (const T&) {                                                    \
      _ok = true;                                                           \
    } catch (...) {                                                         \
    }                                                                       \
    if (!_ok) {                                                             \
      ++g_fail;                                                             \
      std::printf("  FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
    }                                                                       \
  } while (0)

static LigandInstance load(const char* name) {
  std::ifstream in(g_data + "/" + name);
  std::ostringstream b;
  b << in.rdbuf();
  LigandInstance li = parse_instance(b.str());
  li.name = name;
  return li;
}

static LigandInstance single_well() {  // test_docking.cpp:31-37
  LigandInstance inst;
  inst.atoms.push_back({{1.5, 0.0, 0.0}, 1.0, -1});
  inst.sites.push_back({{0.0, 0.0, 0.0}, 1.25, 1.5});
  return inst;
}

static Genotype random_pose(RngStream& rng, int nrot, double spread) {
  Genotype g;
  g.x = rng.uniform(-spread, spread);
  g.y = rng.uniform(-spread, spread);
  g.z = rng.uniform(-spread, spread);
  g.phi = rng.uniform(-3.1, 3.1);
  g.theta = rng.uniform(-3.1, 3.1);
  g.alpha = rng.uniform(-3.1, 3.1);
  for (int k = 0; k < nrot; ++k) g.torsions.push_back(rng.uniform(-3.1, 3.1));
  return g;
}

static LigandInstance random_instance(RngStream& rng, int nrot, int natoms, int nsites) {
  LigandInstance inst;
  inst.n_rot = nrot;
  for (int i = 0; i < natoms; ++i) {
    Atom a;
    a.pos = {rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5)};
    a.weight = rng.uniform(0.5, 1.5);
    a.torsion = nrot > 0 && i % 2 == 0 ? static_cast<int>(rng.next_index(static_cast<std::size_t>(nrot))) : -1;
    inst.atoms.push_back(a);
  }
  for (int i = 0; i < nsites; ++i) {
    Site s;
    s.pos = {rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0), rng.uniform(-2.0, 2.0)};
    s.depth = rng.uniform(0.8, 1.6);
    s.preferred_distance = rng.uniform(1.0, 2.0);
    inst.sites.push_back(s);
  }
  return inst;
}

static void half_frozen() {
  CHECK(f32_to_half(1.0f).bits() == 0x3C00);
  CHECK(f32_to_half(0.1f).bits() == 0x2E66);
  CHECK(f32_to_half(65520.0f).bits() == kHalfPosInf);
  CHECK(f32_to_half(65504.0f).bits() == 0x7BFF);
  CHECK(f32_to_half(std::ldexp(1.0f, -24)).bits() == 0x0001);
  CHECK(f32_to_half(std::ldexp(1.0f, -25)).bits() == 0x0000);
  CHECK(f32_to_half(std::numeric_limits<float>::quiet_NaN()).bits() == kHalfQuietNan);
  CHECK(half_to_f32(Half::from_bits(0x3C00)) == 1.0f);
  CHECK(half_add(f32_to_half(1.0f), f32_to_half(2.0f)).bits() == f32_to_half(3.0f).bits());
}

static void mma_frozen() {
  std::vector<Half> iota(256), id(256, Half()), ones(256, f32_to_half(1.0f));
  for (int i = 0; i < 256; ++i) iota[i] = f32_to_half(static_cast<float>(i));
  for (int i = 0; i < 16; ++i) id[i * 16 + i] = f32_to_half(1.0f);
  const Accum16 d = mma(load_matrix(id, Layout::RowMajor), load_matrix(iota, Layout::RowMajor), Accum16::zero(AccumMode::Single));
  bool ok = true;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) ok = ok && d.at(i, j) == static_cast<float>(i * 16 + j);
  CHECK(ok);
  const Accum16 o = mma(load_matrix(ones, Layout::RowMajor), load_matrix(ones, Layout::RowMajor), Accum16::zero(AccumMode::Half));
  CHECK(o.at(3, 7) == 16.0f);
  CHECK_THROWS_AS(load_matrix(std::vector<Half>(255), Layout::RowMajor), SizeError);
}

static void reduce_frozen() {  // test_reduce.cpp:105-140, 228-342
  std::vector<Vec4> a(64, Vec4{1.0f, 0.0f, 0.0f, 0.0f});
  for (AccumMode m : {AccumMode::Half, AccumMode::Single}) {
    const auto [r, st] = reduce4(a, m);
    CHECK(r.x == 64.0f && r.y == 0.0f && r.e == 0.0f);
    CHECK(st.block_syncs == 2 && st.mma_ops == 2 && st.atomic_adds == 0 && st.memory_fences == 0);
  }
  std::vector<Vec4> b(128);
  for (int i = 0; i < 128; ++i) b[static_cast<std::size_t>(i)] = {static_cast<float>(i % 2), 0.0f, 0.0f, 1.0f};
  const auto [rb, stb] = reduce4(b, AccumMode::Half);
  CHECK(rb.x == 64.0f && rb.e == 128.0f && stb.mma_ops == 3);
  CHECK_THROWS_AS(reduce4(std::vector<Vec4>{}, AccumMode::Half), SizeError);
  std::vector<float> lanes(32);
  for (int i = 0; i < 32; ++i) lanes[static_cast<std::size_t>(i)] = static_cast<float>(i);
  const auto [ws, wst] = baseline_warp_reduce(lanes);
  CHECK(ws == 496.0f && wst.warp_shuffles == 160);
  std::vector<float> idx(1024);
  for (int i = 0; i < 1024; ++i) idx[static_cast<std::size_t>(i)] = static_cast<float>(i);
  const auto [bs, bst] = baseline_block_reduce(idx, 1024);
  CHECK(bs == 523776.0f && bst.atomic_adds == 32 && bst.block_syncs == 3);
  CHECK_THROWS_AS(baseline_block_reduce(std::vector<float>(33), 33), UnsupportedBlockSizeError);
  CHECK_THROWS_AS(baseline_block_reduce(std::vector<float>(64, 1.0f), 96), SizeError);
  std::vector<Partial7> recs(64, Partial7{1, 2, 3, 4, 5, 6, 7});
  for (ReduceMethod m : {ReduceMethod::Baseline, ReduceMethod::Tcu, ReduceMethod::TcuSplit}) {
    const auto [s, st] = reduce7(recs, m, AccumMode::Half);
    CHECK(s[0] == 64.0f && s[1] == 128.0f && s[3] == 256.0f && s[6] == 448.0f);
  }
  CHECK(reduce7(recs, ReduceMethod::Baseline, AccumMode::Half).second.block_syncs == 21);
  CHECK(reduce7(recs, ReduceMethod::Baseline, AccumMode::Half).second.atomic_adds == 14);
  CHECK(reduce7(recs, ReduceMethod::Tcu, AccumMode::Half).second.block_syncs == 4);
  CHECK(reduce7(recs, ReduceMethod::Tcu, AccumMode::Half).second.mma_ops == 4);
  CHECK_THROWS_AS(reduce7(std::vector<Partial7>(63), ReduceMethod::Tcu, AccumMode::Half), UnsupportedBlockSizeError);
  CHECK_THROWS_AS(reduce7(std::vector<Partial7>(63), ReduceMethod::Baseline, AccumMode::Half),
                  UnsupportedBlockSizeError);
}

static void docking_scenarios() {
  // stationarity at d0 (test_docking.cpp:92-118)
  const LigandInstance w = single_well();
  for (auto [m, a] : {std::pair{ReduceMethod::Baseline, AccumMode::Single}, std::pair{ReduceMethod::Tcu, AccumMode::Half}}) {
    const ScoreResult r = score(w, Genotype{}, m, a, 64);
    bool zero = r.energy == -1.25f;
    for (float g : r.gradient) zero = zero && g == 0.0f;
    CHECK(zero);
  }
  CHECK(score_reference(w, Genotype{}).energy == -1.25);
  // validation (test_docking.cpp:120-131)
  CHECK_THROWS_AS(score(w, Genotype{}, ReduceMethod::Tcu, AccumMode::Half, 32), UnsupportedBlockSizeError);
  Genotype wrong;
  wrong.torsions.assign(2, 0.0);
  CHECK_THROWS_AS(score(w, wrong, ReduceMethod::Baseline, AccumMode::Single, 64), SizeError);
  // stats ride along (test_docking.cpp:133-149)
  const LigandInstance s2 = load("s2.mdri");
  RngStream rng = derive_rng(6001, "dock-stats");
  const Genotype g = random_pose(rng, s2.n_rot, 0.5);
  const ScoreResult tcu = score(s2, g, ReduceMethod::Tcu, AccumMode::Half, 64);
  CHECK(tcu.reduce_stats.block_syncs == 4 && tcu.reduce_stats.mma_ops == 4);
  const ScoreResult base = score(s2, g, ReduceMethod::Baseline, AccumMode::Single, 64);
  CHECK(base.reduce_stats.block_syncs == 21 && base.reduce_stats.atomic_adds == 14);
  // FD gradient of the double reference (test_docking.cpp:151-164)
  RngStream fr = derive_rng(6002, "dock-fd");
  const LigandInstance inst = random_instance(fr, 3, 7, 4);
  double worst = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    const Genotype p = random_pose(fr, inst.n_rot, 1.0);
    const RefScore ref = score_reference(inst, p);
    for (int d = 0; d < p.dim(); ++d) {
      Genotype lo = p, hi = p;
      lo.set(d, p.get(d) - 1e-4);
      hi.set(d, p.get(d) + 1e-4);
      const double fd = (score_reference(inst, hi).energy - score_reference(inst, lo).energy) / 2e-4;
      worst = std::max(worst, std::abs(ref.gradient[static_cast<std::size_t>(d)] - fd) / std::max(std::abs(fd), 1.0));
    }
  }
  CHECK(worst < 1e-4);
  // baseline vs tcu single (test_docking.cpp:166-181)
  RngStream xr = derive_rng(6003, "dock-xmethod");
  for (int rep = 0; rep < 25; ++rep) {
    const Genotype p = random_pose(xr, s2.n_rot, 0.35);
    const double ea = score(s2, p, ReduceMethod::Baseline, AccumMode::Single, 64).energy;
    const double eb = score(s2, p, ReduceMethod::Tcu, AccumMode::Single, 64).energy;
    CHECK(std::abs(ea - eb) / std::max({std::abs(ea), std::abs(eb), 0.5}) < 1e-3);
  }
  // ADADELTA first step (test_docking.cpp:211-243)
  std::vector<double> grad(6, 0.0);
  grad[0] = 1.0;
  const auto [st1, g1] = adadelta_step(AdadeltaState::fresh(6), Genotype{}, grad);
  CHECK(std::abs(g1.x - -0.004472091234310839) < 1e-12 * 0.0045);
  CHECK(std::abs(st1.avg_sq_grad[0] - 0.05) < 1e-14);
  std::vector<double> bad(6, 0.0);
  bad[3] = std::numeric_limits<double>::infinity();
  CHECK_THROWS_AS(adadelta_step(AdadeltaState::fresh(6), Genotype{}, bad), NumericDomainError);
  // local search (test_docking.cpp:245-278)
  const LocalSearchResult ls = local_search(w, Genotype{}, 100, 1e-6, ReduceMethod::Tcu, AccumMode::Half, 64, 1);
  CHECK(ls.converged && ls.iterations <= 17 && ls.energy == -1.25 && ls.genotype == Genotype{});
  const LigandInstance s1 = load("s1.mdri");
  RngStream dr = derive_rng(6005, "dock-det");
  const Genotype start = random_pose(dr, s1.n_rot, 0.6);
  CHECK(local_search(s1, start, 80, 1e-4, ReduceMethod::Tcu, AccumMode::Half, 64, 7) ==
        local_search(s1, start, 80, 1e-4, ReduceMethod::Tcu, AccumMode::Half, 64, 7));
  // LGA (test_docking.cpp:280-327)
  LgaSettings cfg;
  cfg.population_size = 8;
  cfg.generations = 2;
  cfg.ls_max_iters = 30;
  const DockResult a = lga_run(s1, ReduceMethod::Tcu, AccumMode::Half, cfg, 4242);
  const DockResult b = lga_run(s1, ReduceMethod::Tcu, AccumMode::Half, cfg, 4242);
  CHECK(a == b && a.evaluations <= cfg.max_evaluations && !a.runs.empty());
  LgaSettings deg;
  deg.population_size = 2;
  deg.generations = 1;
  deg.mutation_sigma = 0.0;
  deg.ls_fraction = 1.0;
  deg.ls_max_iters = 60;
  const DockResult d = lga_run(s1, ReduceMethod::Baseline, AccumMode::Single, deg, 99);
  double best = std::numeric_limits<double>::max();
  for (const LsRunRecord& r : d.runs) best = std::min(best, r.best_energy);
  CHECK(d.runs.size() == 2 && d.best_energy == best);
  LgaSettings tiny;
  tiny.population_size = 1;
  CHECK_THROWS_AS(lga_run(s1, ReduceMethod::Baseline, AccumMode::Single, tiny, 1), SizeError);
  LgaSettings budget;
  budget.population_size = 6;
  budget.generations = 50;
  budget.max_evaluations = 200;
  budget.ls_max_iters = 40;
  CHECK(lga_run(s1, ReduceMethod::Baseline, AccumMode::Single, budget, 7).evaluations <= 200);
  LgaSettings vs;
  vs.population_size = 6;
  vs.generations = 2;
  vs.ls_max_iters = 25;
  const ValidationReport rep = validate_pair(s1, ReduceMethod::Baseline, ReduceMethod::Baseline, AccumMode::Single, 3, 1000, vs);
  CHECK(rep.n_runs == 3 && rep.abs_diff_means == 0.0 && rep.relative_error == 0.0);
  // acceptance.cpp:128-145 on the GPU: paired tcu-half vs baseline, 100 runs
  const ValidationReport pv = validate_pair(s2, ReduceMethod::Baseline, ReduceMethod::Tcu, AccumMode::Half, 100, 12345,
                                            LgaSettings{});
  CHECK(pv.relative_error < 0.002);
  // reference golden: s2, seed 12345, Baseline, default settings
  const DockResult gold = lga_run(s2, ReduceMethod::Baseline, AccumMode::Single, LgaSettings{}, 12345);
  CHECK(gold.best_energy == -10.292128562927246 && gold.evaluations == 27572 && gold.runs.size() == 181);
}

// simblock / instance_io surface (test_simblock.cpp, test_cli.cpp:163-164,
// test_rng_io.cpp CSV cases).
static void simblock_and_csv() {
  const auto rows = scaling_sweep(kDefaultSweepSizes, CostWeights{}, AccumMode::Half);
  const double want[5] = {10.1666667, 15.7727273, 22.5, 28.9347826, 33.8846154};
  CHECK(rows.size() == 5);
  for (int i = 0; i < 5; ++i) CHECK(std::abs(rows[static_cast<std::size_t>(i)].cost_ratio - want[i]) < 1e-6);
  std::vector<Vec4> v(128);
  for (int i = 0; i < 128; ++i) v[static_cast<std::size_t>(i)] = {float(i % 5), 1.0f, float(i % 3) - 1.0f, 0.5f};
  const auto t = simulate_block(BlockConfig(128, ReduceMethod::Tcu, AccumMode::Single), v);
  const auto d = reduce4(v, AccumMode::Single);
  CHECK(t.first.x == d.first.x && t.first.e == d.first.e && t.second == d.second);
  const auto b = simulate_block(BlockConfig(128, ReduceMethod::Baseline, AccumMode::Single), v);
  std::vector<float> xs(128);
  for (int i = 0; i < 128; ++i) xs[static_cast<std::size_t>(i)] = v[static_cast<std::size_t>(i)].x;
  CHECK(b.first.x == baseline_block_reduce(xs, 128).first && b.second.block_syncs == 12);
  CHECK_THROWS_AS(simulate_block(BlockConfig(64, ReduceMethod::Tcu, AccumMode::Half), v), SizeError);
  CHECK(estimate_cost(b.second, CostWeights{}) > 0.0);
  ResultRow r;
  r.seed = 7;
  r.method = "baseline";
  r.accum_mode = "single";
  r.instance = "s1, \"quoted\"";
  r.best_energy = -10.296875;
  r.evaluations = 25549;
  r.converged = true;
  r.block_syncs = 21;
  const std::vector<ResultRow> rr = {r, r};
  const std::string csv = write_results(rr);
  CHECK(csv.rfind("seed,method,accum_mode,instance,best_energy,evaluations,converged,block_syncs,atomic_adds,mma_ops\n", 0) == 0);
  CHECK(csv.find("7,baseline,single,\"s1, \"\"quoted\"\"\",-10.296875,25549,true,21,0,0\n") != std::string::npos);
  CHECK(parse_results(csv) == rr);
  CHECK_THROWS_AS(parse_results("bogus\n"), ParseError);
}

// Extensions (mdreduce::b200): grid-map scoring, clustering, screening.
static void extensions() {
  const LigandInstance s3 = load("s3.mdri");
  b200::GridShape shape;
  shape.nx = shape.ny = shape.nz = 33;
  shape.n_types = 2;
  shape.origin = {-6.0, -6.0, -6.0};
  shape.spacing = 0.375;
  b200::ReceptorFields f;
  for (std::size_t j = 0; j < s3.sites.size(); ++j) {
    f.site_charge.push_back(0.1 * static_cast<double>(j) - 0.15);
    f.site_volume.push_back(1.0);
  }
  f.type_depth_scale = {1.0, 0.7};
  f.type_dist_scale = {1.0, 1.1};
  const b200::Receptor rec = b200::Receptor::build(s3, f, shape);
  const b200::GridMaps maps = rec.download();
  CHECK(maps.maps.size() == 4u * 33 * 33 * 33);
  const b200::Receptor rec2 = b200::Receptor::upload(maps);  // round trip
  b200::LigandChemistry ch;
  for (std::size_t i = 0; i < s3.atoms.size(); ++i) {
    ch.atom_type.push_back(static_cast<int>(i % 2));
    ch.charge.push_back(i % 3 == 0 ? 0.2 : -0.1);
    ch.radius.push_back(0.45);
    ch.epsilon.push_back(0.05);
  }
  Genotype g;
  g.torsions.assign(static_cast<std::size_t>(s3.n_rot), 0.3);
  g.x = 0.4;
  g.phi = 0.2;
  const auto a = b200::grid_score_batch(rec, s3, ch, {g}, ReduceMethod::Baseline, 64);
  const auto b = b200::grid_score_batch(rec2, s3, ch, {g}, ReduceMethod::TcuSplit, 64);
  CHECK(a.size() == 1 && std::isfinite(a[0].energy) && a[0].gradient.size() == 14u);
  CHECK(std::abs(a[0].energy - b[0].energy) <= 1e-5f * std::max(1.0f, std::abs(a[0].energy)));
  CHECK_THROWS_AS(b200::grid_score_batch(rec, s3, ch, {g}, ReduceMethod::Baseline, 16), UnsupportedBlockSizeError);
  LgaSettings st;
  st.generations = 2;
  const auto runs = b200::grid_lga_run_batch(rec, s3, ch, ReduceMethod::Baseline, st, {1, 2, 3, 4});
  CHECK(runs.size() == 4 && runs[0].evaluations > 0 && runs[0].best_energy <= runs[0].runs.back().best_energy);
  std::vector<Genotype> poses;
  std::vector<double> energies;
  for (const DockResult& r : runs) {
    poses.push_back(r.best_genotype);
    energies.push_back(r.best_energy);
  }
  const b200::Clustering c = b200::cluster_poses(s3, poses, energies, 2.0);
  CHECK(c.n_clusters >= 1 && c.n_clusters <= 4 && c.cluster_of.size() == 4u);
  const auto xyz = b200::pose_coordinates(s3, poses[0]);
  CHECK(xyz.size() == s3.atoms.size());
  const auto scr = b200::screen_batch(rec, {s3, s3}, {ch, ch}, 4, ReduceMethod::Baseline, st,
                                      {1, 2, 3, 4, 1, 2, 3, 4}, 2.0);
  CHECK(scr.size() == 2 && scr[0].best_energy == scr[1].best_energy);
  for (int k = 0; k < 4; ++k) CHECK(scr[0].best_energy[static_cast<std::size_t>(k)] == runs[static_cast<std::size_t>(k)].best_energy);
  CHECK(scr[0].clusters.cluster_of == c.cluster_of && scr[0].clusters.n_clusters == c.n_clusters);
  // exact-torsion mode: torsion entries follow score_reference's per-group torque
  b200::set_exact_torsion(true);
  const auto ex = b200::score_batch(s3, {g}, ReduceMethod::Baseline, AccumMode::Single, 64);
  b200::set_exact_torsion(false);
  const auto ap = b200::score_batch(s3, {g}, ReduceMethod::Baseline, AccumMode::Single, 64);
  const RefScore rs = score_reference(s3, g);
  double scale = 1.0, err = 0.0;
  for (double v : rs.gradient) scale = std::max(scale, std::abs(v));
  for (std::size_t d = 6; d < rs.gradient.size(); ++d) err = std::max(err, std::abs(ex[0].gradient[d] - rs.gradient[d]));
  CHECK(err <= 2e-6 * scale);
  CHECK(ex[0].energy == ap[0].energy && ex[0].gradient[3] == ap[0].gradient[3]);
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::printf("usage: %s <data dir>\n", argv[0]);
    return 2;
  }
  g_data = argv[1];
  const std::pair<const char*, std::function<void()>> suites[] = {
      {"half", half_frozen}, {"mma", mma_frozen}, {"reduce", reduce_frozen}, {"docking", docking_scenarios},
      {"simblock+csv", simblock_and_csv}, {"extensions", extensions}};
  for (const auto& [name, fn] : suites) {
    const int before = g_fail;
    fn();
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
  return g_fail == 0 ? 0 : 1;
}
