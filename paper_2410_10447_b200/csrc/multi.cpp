// multi.cpp — native multi-GPU host driver (north_star subsystem 4, SURVEY
// §8 e): one host thread and one mdr context per device of the node.
//
//  * mdr_multi_lga_run_batch: independent LGA runs (validate_pair-style seed
//    lists, docking.cpp:558-564) sharded statically, run i -> device
//    i mod n_devices; every device docks its shard as one CUDA-graph batch;
//  * mdr_multi_screen: ligands pulled from a shared atomic work queue in
//    batches (ligand costs differ by ~100x, so a dynamic queue balances the
//    devices), each batch one mdr_grid_screen_batch launch sequence against
//    the device's own copy of the receptor maps.  Failure handling (SURVEY
//    §5): a device whose batch fails with a device error retires and puts
//    the batch on a retry list that the surviving devices drain; the call
//    fails only if every device has retired (or on a non-device error, e.g.
//    a ligand the path rejects).  mdr_multi_set_fault_injection(d, k) makes
//    device index d fail on its k-th batch (tests).
// The only exchange is the final gather: every thread writes its results
// into the caller's arrays at the run / ligand's own offsets (no collective,
// no NCCL: the path is embarrassingly parallel).  Results are identical to a
// single-device call on the same seeds (tests/test_multi.py).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "mdr.h"

namespace {

struct CtxGuard {
  mdr_ctx* c = nullptr;
  ~CtxGuard() {
    if (c) mdr_ctx_destroy(c);
  }
};

std::atomic<int> g_fault_device{-1}, g_fault_batch{0};

struct FirstError {  // the first failure of any device thread wins
  std::mutex m;
  std::atomic<int> rc{MDR_OK};
  std::string msg;
  void set(int code, const char* what) {
    std::lock_guard<std::mutex> g(m);
    if (rc.load() == MDR_OK) {
      msg = what ? what : "";
      rc.store(code);
    }
  }
};

thread_local std::string t_multi_err;

int finish(FirstError& fe) {
  if (fe.rc != MDR_OK) t_multi_err = fe.msg;
  return fe.rc;
}

}  // namespace

extern "C" {

const char* mdr_multi_last_error(void) { return t_multi_err.c_str(); }

void mdr_multi_set_fault_injection(int device_index, int batch) {
  g_fault_device.store(device_index);
  g_fault_batch.store(batch);
}

int mdr_multi_lga_run_batch(const int* devices, int n_devices, const mdr_instance* inst, int method, int accum,
                            int pair_precision, const mdr_lga_settings* s, const uint64_t* seeds, int n_runs,
                            double* best_energy, double* best_genotype, int64_t* evaluations, int32_t* converged) {
  if (!devices || n_devices < 1 || !inst || !s || n_runs < 0 || (n_runs && !seeds)) return MDR_ERR_INVALID;
  if (n_runs == 0) return MDR_OK;
  const int dim = 6 + inst->n_rot;
  FirstError fe;
  std::vector<std::thread> pool;
  for (int t = 0; t < n_devices; ++t) {
    pool.emplace_back([&, t] {
      std::vector<int> mine;
      for (int i = t; i < n_runs; i += n_devices) mine.push_back(i);
      if (mine.empty()) return;
      CtxGuard g;
      g.c = mdr_ctx_create(devices[t]);
      if (!g.c) return fe.set(MDR_ERR_CUDA, "mdr_ctx_create failed");
      if (int rc = mdr_ctx_set_pair_precision(g.c, pair_precision)) return fe.set(rc, mdr_last_error(g.c));
      const int n = (int)mine.size();
      std::vector<uint64_t> sd(n);
      for (int k = 0; k < n; ++k) sd[k] = seeds[mine[k]];
      std::vector<double> be(n), bg((size_t)n * dim);
      std::vector<int64_t> ev(n);
      std::vector<int32_t> cv(n), nr(n);
      std::vector<mdr_ls_record> recs((size_t)n * mdr_lga_max_records(s));
      const int rc = mdr_lga_run_batch(g.c, inst, method, accum, s, sd.data(), n, be.data(), bg.data(), ev.data(),
                                       cv.data(), nr.data(), recs.data(), nullptr);
      if (rc) return fe.set(rc, mdr_last_error(g.c));
      for (int k = 0; k < n; ++k) {  // gather by run index
        const int i = mine[k];
        if (best_energy) best_energy[i] = be[k];
        if (best_genotype) std::memcpy(best_genotype + (size_t)i * dim, &bg[(size_t)k * dim], sizeof(double) * dim);
        if (evaluations) evaluations[i] = ev[k];
        if (converged) converged[i] = cv[k];
      }
    });
  }
  for (auto& th : pool) th.join();
  return finish(fe);
}

int mdr_multi_screen(const int* devices, int n_devices, const mdr_instance* receptor_sites,
                     const mdr_receptor_fields* fields, const mdr_grid* shape, const mdr_instance* ligands,
                     const mdr_ligand_params* params, int n_ligands, int runs_per_ligand, int method,
                     const mdr_lga_settings* s, const uint64_t* seeds, double rmsd_tol, int batch_ligands,
                     double* best_energy, double* best_genotype, int64_t* evaluations, int32_t* cluster_of,
                     int32_t* n_clusters, int32_t* device_of_ligand) {
  if (!devices || n_devices < 1 || !receptor_sites || !fields || !shape || !ligands || !params || !s ||
      n_ligands < 0 || runs_per_ligand < 0 || batch_ligands < 1 || (n_ligands && runs_per_ligand && !seeds))
    return MDR_ERR_INVALID;
  if (n_ligands == 0 || runs_per_ligand == 0) return MDR_OK;
  const int R = runs_per_ligand;
  // genotype offsets of each ligand in the packed best_genotype output
  std::vector<size_t> goff(n_ligands + 1, 0);
  for (int j = 0; j < n_ligands; ++j) goff[j + 1] = goff[j] + (size_t)R * (6 + ligands[j].n_rot);
  // Work queue: fresh batches in order, then batches handed back by retired
  // devices.  A device leaves only when nothing is queued and no batch is in
  // flight anywhere (an in-flight batch may still come back).
  std::mutex qm;
  int next_j = 0, busy = 0;
  std::vector<int> retry;
  FirstError fe;
  auto acquire = [&]() -> int {
    for (;;) {
      {
        std::lock_guard<std::mutex> g(qm);
        if (fe.rc != MDR_OK) return -1;
        if (next_j < n_ligands) {
          const int j = next_j;
          next_j += batch_ligands;
          ++busy;
          return j;
        }
        if (!retry.empty()) {
          const int j = retry.back();
          retry.pop_back();
          ++busy;
          return j;
        }
        if (busy == 0) return -1;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  };
  auto release = [&](int handed_back) {
    std::lock_guard<std::mutex> g(qm);
    if (handed_back >= 0) retry.push_back(handed_back);
    --busy;
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < n_devices; ++t) {
    pool.emplace_back([&, t] {
      CtxGuard g;
      g.c = mdr_ctx_create(devices[t]);
      if (!g.c) return;  // this device never takes work
      mdr_dev_grid* dg = mdr_grid_build(g.c, receptor_sites, fields, shape);  // receptor once per device
      if (!dg) return;
      int done = 0;
      for (;;) {
        const int j0 = acquire();
        if (j0 < 0) break;
        const int nb = std::min(batch_ligands, n_ligands - j0);
        std::vector<double> be((size_t)nb * R), bg(goff[j0 + nb] - goff[j0]);
        std::vector<int64_t> ev((size_t)nb * R);
        std::vector<int32_t> cl((size_t)nb * R), nc(nb), cv((size_t)nb * R);
        const int rc = (g_fault_device.load() == t && done == g_fault_batch.load())
                           ? MDR_ERR_CUDA  // injected device failure
                           : mdr_grid_screen_batch(g.c, dg, ligands + j0, params + j0, nb, R, method, s,
                                                   seeds + (size_t)j0 * R, rmsd_tol, be.data(), bg.data(),
                                                   ev.data(), cv.data(), cl.data(), nullptr, nc.data());
        if (rc == MDR_ERR_CUDA) {  // device failure: hand the batch back and retire
          release(j0);
          break;
        }
        if (rc) {  // the batch itself is invalid: no device would succeed
          fe.set(rc, mdr_last_error(g.c));
          release(-1);
          break;
        }
        ++done;
        const size_t r0 = (size_t)j0 * R;
        if (best_energy) std::memcpy(best_energy + r0, be.data(), sizeof(double) * be.size());
        if (best_genotype) std::memcpy(best_genotype + goff[j0], bg.data(), sizeof(double) * bg.size());
        if (evaluations) std::memcpy(evaluations + r0, ev.data(), sizeof(int64_t) * ev.size());
        if (cluster_of) std::memcpy(cluster_of + r0, cl.data(), sizeof(int32_t) * cl.size());
        if (n_clusters) std::memcpy(n_clusters + j0, nc.data(), sizeof(int32_t) * nb);
        if (device_of_ligand)
          for (int k = 0; k < nb; ++k) device_of_ligand[j0 + k] = t;
        release(-1);
      }
      mdr_grid_free(g.c, dg);
    });
  }
  for (auto& th : pool) th.join();
  if (fe.rc == MDR_OK && (!retry.empty() || next_j < n_ligands))
    fe.set(MDR_ERR_CUDA, "every device failed; batches left undocked");
  return finish(fe);
}

}  // extern "C"
