// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never shipped).
//
// A flat C-ABI over the UNMODIFIED reference library, compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libmdr_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's CPU arm may load it.
// Every function forwards to the reference's own C++ API (namespace mdreduce)
// and converts its exceptions into the status codes of include/mdr.h.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mdr.h"
#include "mdreduce/docking.hpp"
#include "mdreduce/errors.hpp"
#include "mdreduce/half.hpp"
#include "mdreduce/instance_io.hpp"
#include "mdreduce/mma.hpp"
#include "mdreduce/reduce.hpp"
#include "mdreduce/rng.hpp"
#include "mdreduce/simblock.hpp"

using namespace mdreduce;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return MDR_OK;
    } catch (const SizeError& e) {
        g_err = e.what();
        return MDR_ERR_SIZE;
    } catch (const UnsupportedBlockSizeError& e) {
        g_err = e.what();
        return MDR_ERR_BLOCK_SIZE;
    } catch (const NumericDomainError& e) {
        g_err = e.what();
        return MDR_ERR_NUMERIC_DOMAIN;
    } catch (const ParseError& e) {
        g_err = e.what();
        return MDR_ERR_PARSE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MDR_ERR_INVALID;
    }
}

LigandInstance to_inst(const mdr_instance* in) {
    LigandInstance li;
    li.n_rot = in->n_rot;
    for (int i = 0; i < in->n_atoms; ++i) {
        Atom a;
        a.pos = {in->atom_xyzw[4 * i], in->atom_xyzw[4 * i + 1], in->atom_xyzw[4 * i + 2]};
        a.weight = in->atom_xyzw[4 * i + 3];
        a.torsion = in->atom_torsion[i];
        li.atoms.push_back(a);
    }
    for (int i = 0; i < in->n_sites; ++i) {
        Site s;
        s.pos = {in->site_xyzdd[5 * i], in->site_xyzdd[5 * i + 1], in->site_xyzdd[5 * i + 2]};
        s.depth = in->site_xyzdd[5 * i + 3];
        s.preferred_distance = in->site_xyzdd[5 * i + 4];
        li.sites.push_back(s);
    }
    return li;
}

Genotype to_geno(const double* g, int n_rot) {
    Genotype out;
    out.torsions.resize(static_cast<std::size_t>(n_rot));
    for (int d = 0; d < 6 + n_rot; ++d) out.set(d, g[d]);
    return out;
}

void from_geno(const Genotype& g, double* out) {
    for (int d = 0; d < g.dim(); ++d) out[d] = g.get(d);
}

void put_stats(const SyncStats& s, mdr_sync_stats* o) {
    if (!o) return;
    o->block_syncs = s.block_syncs;
    o->warp_shuffles = s.warp_shuffles;
    o->atomic_adds = s.atomic_adds;
    o->memory_fences = s.memory_fences;
    o->mma_ops = s.mma_ops;
    o->shared_mem_bytes = s.shared_mem_bytes;
    o->precision_conversions = s.precision_conversions;
}

ReduceMethod meth(int m) { return m == MDR_METHOD_TCU ? ReduceMethod::Tcu : ReduceMethod::Baseline; }
AccumMode acc(int a) { return a == MDR_ACCUM_SINGLE ? AccumMode::Single : AccumMode::Half; }

LgaSettings to_settings(const mdr_lga_settings* s) {
    LgaSettings o;
    o.population_size = s->population_size;
    o.generations = s->generations;
    o.max_evaluations = s->max_evaluations;
    o.ls_fraction = s->ls_fraction;
    o.ls_max_iters = s->ls_max_iters;
    o.ls_convergence_tol = s->ls_convergence_tol;
    o.mutation_sigma = s->mutation_sigma;
    o.partition = s->partition;
    return o;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rng_draws(uint64_t seed, const char* label, uint64_t n, uint64_t* out) {
    RngStream r = derive_rng(seed, label);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void ref_rng_normals(uint64_t seed, const char* label, uint64_t n, double* out) {
    RngStream r = derive_rng(seed, label);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
}

void ref_f32_to_half(const float* in, size_t n, uint16_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = f32_to_half(in[i]).bits();
}

void ref_half_to_f32(const uint16_t* in, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = half_to_f32(Half::from_bits(in[i]));
}

int ref_mma(const uint16_t* a, const uint16_t* b, const float* c, int accum, float* d) {
    return guarded([&] {
        std::vector<Half> av(256), bv(256);
        for (int i = 0; i < 256; ++i) {
            av[i] = Half::from_bits(a[i]);
            bv[i] = Half::from_bits(b[i]);
        }
        const Mat16 A = load_matrix(av, Layout::RowMajor);
        const Mat16 B = load_matrix(bv, Layout::RowMajor);
        Accum16 C(acc(accum));
        for (int i = 0; i < 16; ++i)
            for (int j = 0; j < 16; ++j) C.set(i, j, c[i * 16 + j]);
        const Accum16 D = mma(A, B, C);
        const std::vector<float> out = store_matrix(D, Layout::RowMajor);
        std::memcpy(d, out.data(), 256 * sizeof(float));
    });
}

int ref_reduce4(const float* vecs, int n, int accum, float* out, mdr_sync_stats* st) {
    return guarded([&] {
        std::vector<Vec4> v(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) v[i] = Vec4{vecs[4 * i], vecs[4 * i + 1], vecs[4 * i + 2], vecs[4 * i + 3]};
        auto [r, s] = reduce4(v, acc(accum));
        out[0] = r.x;
        out[1] = r.y;
        out[2] = r.z;
        out[3] = r.e;
        put_stats(s, st);
    });
}

int ref_simulate_block4(const float* vecs, int n, int method, int accum, float* out,
                        mdr_sync_stats* st) {
    return guarded([&] {
        std::vector<Vec4> v(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) v[i] = Vec4{vecs[4 * i], vecs[4 * i + 1], vecs[4 * i + 2], vecs[4 * i + 3]};
        const BlockConfig cfg(n, meth(method), acc(accum));
        auto [r, s] = simulate_block(cfg, std::span<const Vec4>(v));
        out[0] = r.x;
        out[1] = r.y;
        out[2] = r.z;
        out[3] = r.e;
        put_stats(s, st);
    });
}

int ref_warp_reduce(const float* lanes, int n, float* out, mdr_sync_stats* st) {
    return guarded([&] {
        auto [r, s] = baseline_warp_reduce(std::span<const float>(lanes, static_cast<std::size_t>(n)));
        *out = r;
        put_stats(s, st);
    });
}

int ref_block_reduce(const float* values, int n, int threads, float* out, mdr_sync_stats* st) {
    return guarded([&] {
        auto [r, s] = baseline_block_reduce(std::span<const float>(values, static_cast<std::size_t>(n)), threads);
        *out = r;
        put_stats(s, st);
    });
}

int ref_reduce7(const float* recs, int n, int method, int accum, float* out, mdr_sync_stats* st) {
    return guarded([&] {
        std::vector<Partial7> v(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            const float* r = recs + 7 * i;
            v[i] = Partial7{r[0], r[1], r[2], r[3], r[4], r[5], r[6]};
        }
        auto [r, s] = reduce7(v, meth(method), acc(accum));
        for (int c = 0; c < 7; ++c) out[c] = r[static_cast<std::size_t>(c)];
        put_stats(s, st);
    });
}

int ref_score(const mdr_instance* inst, const double* g, int method, int accum, int partition,
              float* energy, float* grad, float* torque, mdr_sync_stats* st) {
    return guarded([&] {
        const LigandInstance li = to_inst(inst);
        const ScoreResult r = score(li, to_geno(g, inst->n_rot), meth(method), acc(accum), partition);
        *energy = r.energy;
        for (std::size_t d = 0; d < r.gradient.size(); ++d) grad[d] = r.gradient[d];
        for (int c = 0; c < 3; ++c) torque[c] = r.torque[static_cast<std::size_t>(c)];
        put_stats(r.reduce_stats, st);
    });
}

// Batched score over a shared instance (avoids re-converting the instance).
int ref_score_many(const mdr_instance* inst, const double* gs, int n, int method, int accum,
                   int partition, float* energy, float* grad, float* torque) {
    return guarded([&] {
        const LigandInstance li = to_inst(inst);
        const int dim = 6 + inst->n_rot;
        for (int i = 0; i < n; ++i) {
            const ScoreResult r = score(li, to_geno(gs + i * dim, inst->n_rot), meth(method),
                                        acc(accum), partition);
            energy[i] = r.energy;
            for (int d = 0; d < dim; ++d) grad[i * dim + d] = r.gradient[static_cast<std::size_t>(d)];
            for (int c = 0; c < 3; ++c) torque[i * 3 + c] = r.torque[static_cast<std::size_t>(c)];
        }
    });
}

int ref_score_reference(const mdr_instance* inst, const double* g, double* energy, double* grad,
                        double* torque) {
    return guarded([&] {
        const RefScore r = score_reference(to_inst(inst), to_geno(g, inst->n_rot));
        *energy = r.energy;
        for (std::size_t d = 0; d < r.gradient.size(); ++d) grad[d] = r.gradient[d];
        for (int c = 0; c < 3; ++c) torque[c] = r.torque[static_cast<std::size_t>(c)];
    });
}

int ref_adadelta_step(int dim, double rho, double eps, double* avg_sq_grad, double* avg_sq_update,
                      double* genotype, const double* grad) {
    return guarded([&] {
        AdadeltaState s;
        s.avg_sq_grad.assign(avg_sq_grad, avg_sq_grad + dim);
        s.avg_sq_update.assign(avg_sq_update, avg_sq_update + dim);
        s.rho = rho;
        s.epsilon = eps;
        const Genotype g = to_geno(genotype, dim - 6);
        auto [ns, ng] = adadelta_step(s, g, std::vector<double>(grad, grad + dim));
        std::memcpy(avg_sq_grad, ns.avg_sq_grad.data(), sizeof(double) * dim);
        std::memcpy(avg_sq_update, ns.avg_sq_update.data(), sizeof(double) * dim);
        from_geno(ng, genotype);
    });
}

int ref_local_search(const mdr_instance* inst, const double* start, int max_iters, double tol,
                     int method, int accum, int partition, double* out_g, double* out_e,
                     int32_t* out_iters, int32_t* out_conv, mdr_sync_stats* st) {
    return guarded([&] {
        const LocalSearchResult r = local_search(to_inst(inst), to_geno(start, inst->n_rot), max_iters,
                                                 tol, meth(method), acc(accum), partition, 0);
        from_geno(r.genotype, out_g);
        *out_e = r.energy;
        *out_iters = r.iterations;
        *out_conv = r.converged ? 1 : 0;
        put_stats(r.stats, st);
    });
}

int ref_lga_run(const mdr_instance* inst, int method, int accum, const mdr_lga_settings* s,
                uint64_t seed, double* best_e, double* best_g, int64_t* evals, int32_t* conv,
                int32_t* n_records, mdr_ls_record* records, int max_records, mdr_sync_stats* st) {
    return guarded([&] {
        const DockResult r = lga_run(to_inst(inst), meth(method), acc(accum), to_settings(s), seed);
        *best_e = r.best_energy;
        from_geno(r.best_genotype, best_g);
        *evals = r.evaluations;
        *conv = r.converged ? 1 : 0;
        const int nr = static_cast<int>(r.runs.size());
        *n_records = nr;
        for (int i = 0; i < nr && i < max_records; ++i) {
            records[i].best_energy = r.runs[static_cast<std::size_t>(i)].best_energy;
            records[i].iterations = r.runs[static_cast<std::size_t>(i)].iterations;
            records[i].converged = r.runs[static_cast<std::size_t>(i)].converged ? 1 : 0;
        }
        put_stats(r.total_stats, st);
    });
}

double ref_torsion_axis(int k, double* out3) {
    const auto a = torsion_axis(k);
    out3[0] = a[0];
    out3[1] = a[1];
    out3[2] = a[2];
    return 0.0;
}

// parse_instance instance_io.cpp:137-253 into caller buffers (capacity-checked).
int ref_parse_instance(const char* text, int cap_atoms, int cap_sites, int32_t* n_atoms,
                       int32_t* n_sites, int32_t* n_rot, double* atom_xyzw, int32_t* atom_torsion,
                       double* site_xyzdd, int32_t* err_line) {
    *err_line = 0;
    try {
        const LigandInstance li = parse_instance(text);
        *n_atoms = static_cast<int32_t>(li.atoms.size());
        *n_sites = static_cast<int32_t>(li.sites.size());
        *n_rot = li.n_rot;
        if (*n_atoms > cap_atoms || *n_sites > cap_sites) return MDR_ERR_SIZE;
        for (int i = 0; i < *n_atoms; ++i) {
            const Atom& a = li.atoms[static_cast<std::size_t>(i)];
            atom_xyzw[4 * i] = a.pos[0];
            atom_xyzw[4 * i + 1] = a.pos[1];
            atom_xyzw[4 * i + 2] = a.pos[2];
            atom_xyzw[4 * i + 3] = a.weight;
            atom_torsion[i] = a.torsion;
        }
        for (int i = 0; i < *n_sites; ++i) {
            const Site& s = li.sites[static_cast<std::size_t>(i)];
            site_xyzdd[5 * i] = s.pos[0];
            site_xyzdd[5 * i + 1] = s.pos[1];
            site_xyzdd[5 * i + 2] = s.pos[2];
            site_xyzdd[5 * i + 3] = s.depth;
            site_xyzdd[5 * i + 4] = s.preferred_distance;
        }
        return MDR_OK;
    } catch (const ParseError& e) {
        g_err = e.what();
        *err_line = e.line();
        return MDR_ERR_PARSE;
    }
}

// write_results instance_io.cpp:277-287 over n rows given as parallel
// arrays; the CSV text (NUL-terminated, truncated to cap) goes to out.
int ref_write_results(int n, const uint64_t* seed, const char* const* method, const char* const* accum,
                      const char* const* instance, const double* best_energy, const int64_t* evaluations,
                      const int32_t* converged, const uint64_t* block_syncs, const uint64_t* atomic_adds,
                      const uint64_t* mma_ops, char* out, size_t cap, size_t* len) {
    return guarded([&] {
        std::vector<ResultRow> rows(n);
        for (int i = 0; i < n; ++i) {
            rows[i].seed = seed[i];
            rows[i].method = method[i];
            rows[i].accum_mode = accum[i];
            rows[i].instance = instance[i];
            rows[i].best_energy = best_energy[i];
            rows[i].evaluations = evaluations[i];
            rows[i].converged = converged[i] != 0;
            rows[i].block_syncs = block_syncs[i];
            rows[i].atomic_adds = atomic_adds[i];
            rows[i].mma_ops = mma_ops[i];
        }
        const std::string s = write_results(rows);
        *len = s.size();
        const size_t k = s.size() < cap ? s.size() : cap - 1;
        std::memcpy(out, s.data(), k);
        out[k] = 0;
    });
}

// ---- C2 CPU leg (test / bench infrastructure): the reference's own
// reduction calls timed in a loop, like cli.cpp:195-266 (cmd_reduce_bench).

// out[i] = (float) uniform(-1, 1) of draw i + 1 of derive_rng(seed, label)
// (rng.hpp:41-43, rng.cpp:43-45): the C2 inputs, identical to
// the device generator's.
int ref_fill_uniform(uint64_t seed, const char* label, int64_t n, float* out) {
    return guarded([&] {
        RngStream rng = derive_rng(seed, label);
        for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng.uniform(-1.0, 1.0));
    });
}

// Calls of one reduction over the n_red input sets of B records (cycled)
// until budget_s elapsed; *ns_per_call = wall time / calls.
//   kind 0: reduce4 (reduce.cpp:80-111; in = n_red x B x 4) with
//           method TCU, or simulate_block's baseline four block reductions
//           (simblock.cpp) with method BASELINE;
//   kind 1: reduce7 (reduce.cpp:165-209; in = n_red x B x 7), either method;
//   kind 2: baseline_block_reduce (reduce.cpp:136-163; in = n_red x B).
int ref_time_reduce(int kind, int method, int accum, int B, const float* in, int n_red, double budget_s,
                    double* ns_per_call, double* checksum, int64_t* calls) {
    return guarded([&] {
        const int comps = kind == 0 ? 4 : (kind == 1 ? 7 : 1);
        std::vector<std::vector<Vec4>> v4;
        std::vector<std::vector<Partial7>> v7;
        for (int r = 0; r < n_red; ++r) {
            const float* p = in + static_cast<size_t>(r) * B * comps;
            if (kind == 0) {
                std::vector<Vec4> v(static_cast<size_t>(B));
                for (int t = 0; t < B; ++t) v[t] = Vec4{p[4 * t], p[4 * t + 1], p[4 * t + 2], p[4 * t + 3]};
                v4.push_back(std::move(v));
            } else if (kind == 1) {
                std::vector<Partial7> v(static_cast<size_t>(B));
                for (int t = 0; t < B; ++t)
                    v[t] = Partial7{p[7 * t], p[7 * t + 1], p[7 * t + 2], p[7 * t + 3], p[7 * t + 4], p[7 * t + 5],
                                    p[7 * t + 6]};
                v7.push_back(std::move(v));
            }
        }
        const BlockConfig cfg(B, meth(method), acc(accum));
        double sum = 0.0;
        int64_t n = 0;
        const auto t0 = std::chrono::steady_clock::now();
        double el = 0.0;
        do {
            for (int r = 0; r < n_red; ++r, ++n) {
                if (kind == 0) {
                    if (method == MDR_METHOD_TCU) {
                        auto [x, st] = reduce4(v4[r], acc(accum));
                        sum += x.x;
                    } else {
                        auto [x, st] = simulate_block(cfg, std::span<const Vec4>(v4[r]));
                        sum += x.x;
                    }
                } else if (kind == 1) {
                    auto [x, st] = reduce7(v7[r], meth(method), acc(accum));
                    sum += x[0];
                } else {
                    auto [x, st] = baseline_block_reduce(
                        std::span<const float>(in + static_cast<size_t>(r) * B, static_cast<size_t>(B)), B);
                    sum += x;
                }
            }
            el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        } while (el < budget_s);
        *ns_per_call = el * 1e9 / static_cast<double>(n);
        *checksum = sum;
        *calls = n;
    });
}

} // extern "C"
