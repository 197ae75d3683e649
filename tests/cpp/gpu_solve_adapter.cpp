// SPDX-License-Identifier: Apache-2.0
//
// The drop-in adapter of INTEGRATION.md, compiled against the reference's
// own headers (proj/include/fsi) and the fsigpu C ABI. It is what a
// maintainer adds to the reference tree to replace the solve block of
// FsiSolver::newton_step (proj/src/driver.cpp:257-272). tests/test_abi.py
// syntax-checks it here; oracle/Makefile `adapter` links it with the
// reference library and libfsigpu.so into oracle/_ref/fsi_adapter_check
// (the harness's `gpu-adapter` command), which tests/test_gpu_parity.py
// runs on the GPU against the reference's own gmres.
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsi/driver.hpp"
#include "fsi/errors.hpp"
#include "fsi/gmg.hpp"
#include "fsi/krylov.hpp"
#include "fsi/precond.hpp"
#include "fsigpu.h"

namespace fsi {
namespace {

// Status -> the reference's exceptions. A singular block is named by the
// reference IndexSet label of the failing block (labels[level][block],
// e.g. "fs-fluid-up-12", precond.cpp:182,224,265); non-block failures
// ("gmg-coarse", "fs lumped mass row <i>") come with the message. Device
// faults are NOT SolverError: the driver catches SolverError as a
// non-converged Newton step and retries with dt halved (driver.cpp:369),
// which must not happen on a dead CUDA context.
void check(int rc, const std::map<int, std::vector<std::string>>* labels = nullptr) {
  if (rc == FSIGPU_OK) return;
  const std::string msg = fsigpu_last_error();
  if (rc == FSIGPU_ERR_SINGULAR) {
    const int b = fsigpu_last_singular_block(), l = fsigpu_last_singular_level();
    if (labels && b >= 0) {
      auto it = labels->find(l);
      if (it != labels->end() && b < static_cast<int>(it->second.size())) throw SingularBlockError(it->second[b]);
    }
    const std::string prefix = "singular block: ";
    throw SingularBlockError(msg.compare(0, prefix.size(), prefix) == 0 ? msg.substr(prefix.size()) : msg);
  }
  if (rc == FSIGPU_ERR_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error("fsigpu device failure: " + msg);
}

void flatten(const std::vector<const IndexSet*>& sets, std::vector<int>& ptr, std::vector<int>& idx) {
  ptr.assign(1, 0);
  idx.clear();
  for (const IndexSet* s : sets) {
    idx.insert(idx.end(), s->indices.begin(), s->indices.end());
    ptr.push_back(static_cast<int>(idx.size()));
  }
}

}  // namespace

// GMG with FS smoothers on the GPU, presented as the reference's
// LinearOperator (include/fsi/krylov.hpp:14-18).
class GpuGmg final : public LinearOperator {
 public:
  GpuGmg(const std::vector<GmgLevel>& levels, const std::vector<const FsPreconditioner*>& fs,
         const CycleConfig& cfg) {
    std::vector<fsigpu_level_desc> d(levels.size());
    for (size_t l = 0; l < levels.size(); ++l) {
      const SparseMatrix& a = *levels[l].a;
      fsigpu_level_desc& x = d[l];
      x = fsigpu_level_desc{};
      x.n = a.rows();
      x.a_ptr = a.row_offsets().data();
      x.a_idx = a.col_indices().data();
      x.a_val = a.values().data();
      x.row_mask = levels[l].constrained_rows.data();
      x.col_mask = levels[l].constrained_cols.data();
      if (l == 0) continue;
      x.nc = levels[l].p.cols();
      x.p_ptr = levels[l].p.row_offsets().data();
      x.p_idx = levels[l].p.col_indices().data();
      x.p_val = levels[l].p.values().data();
      x.r_ptr = levels[l].r.row_offsets().data();
      x.r_idx = levels[l].r.col_indices().data();
      x.r_val = levels[l].r.values().data();
      const FsPreconditioner& f = *fs[l];
      x.g1 = f.group1_size();
      x.n_us = f.solid_velocity_size();
      x.lumped = f.lumped().data();
      std::vector<const IndexSet*> s1, s2;
      for (int b = 0; b < f.as1().n_blocks(); ++b) s1.push_back(&f.as1().block_dofs(b));
      for (int b = 0; b < f.n_fluid_blocks(); ++b) s2.push_back(&f.fluid_block_dofs(b));
      for (const IndexSet* is : s1) labels_[static_cast<int>(l)].push_back(is->label);
      for (const IndexSet* is : s2) labels_[static_cast<int>(l)].push_back(is->label);
      flatten(s1, as1_ptr_[l], as1_idx_[l]);
      flatten(s2, as2_ptr_[l], as2_idx_[l]);
      x.as1_n = static_cast<int>(as1_ptr_[l].size()) - 1;
      x.as1_ptr = as1_ptr_[l].data();
      x.as1_idx = as1_idx_[l].data();
      x.as2_n = static_cast<int>(as2_ptr_[l].size()) - 1;
      x.as2_ptr = as2_ptr_[l].data();
      x.as2_idx = as2_idx_[l].data();
    }
    check(fsigpu_gmg_create(static_cast<int>(d.size()), d.data(), cfg.omega, cfg.pre, cfg.post, cfg.cycle, &h_),
          &labels_);
  }
  // The same hierarchy without the reference FsPreconditioner (which
  // factorises every block on the CPU to build itself): the block sets and
  // the lumped mass are built on the GPU from each level's Space, J2
  // OrderingPlan and constraint masks (fsigpu_fs_sets_build, precond.cpp:
  // 119-269), as the driver would pass them (driver.cpp:229-256).
  GpuGmg(const std::vector<GmgLevel>& levels, const std::vector<const Space*>& spaces,
         const std::vector<const OrderingPlan*>& j2, const std::vector<const ConstraintMasks*>& masks,
         const FieldSplitPlan& plan, const CycleConfig& cfg) {
    std::vector<fsigpu_level_desc> d(levels.size());
    for (size_t l = 0; l < levels.size(); ++l) {
      const SparseMatrix& a = *levels[l].a;
      fsigpu_level_desc& x = d[l];
      x = fsigpu_level_desc{};
      x.n = a.rows();
      x.a_ptr = a.row_offsets().data();
      x.a_idx = a.col_indices().data();
      x.a_val = a.values().data();
      x.row_mask = levels[l].constrained_rows.data();
      x.col_mask = levels[l].constrained_cols.data();
      if (l == 0) continue;
      x.nc = levels[l].p.cols();
      x.p_ptr = levels[l].p.row_offsets().data();
      x.p_idx = levels[l].p.col_indices().data();
      x.p_val = levels[l].p.values().data();
      x.r_ptr = levels[l].r.row_offsets().data();
      x.r_idx = levels[l].r.col_indices().data();
      x.r_val = levels[l].r.values().data();
      const OrderingPlan& o = *j2[l];
      x.g1 = o.block_offsets[3];  // precond.cpp:128-130
      x.n_us = o.block_offsets[4] - o.block_offsets[3];
      const Space& sp = *spaces[l];
      const FieldLayout& fl = sp.layout;
      std::vector<int>& en = mesh_[l].en;
      std::vector<int>& dp = mesh_[l].dp;
      std::vector<int>& up = mesh_[l].up;
      std::vector<int>& pp = mesh_[l].pp;
      for (int e = 0; e < fl.n_elements; ++e)
        for (int k = 0; k < 9; ++k) en.push_back(sp.dofmap.element_nodes[e][k]);
      for (int q = 0; q < fl.n_q2_nodes; ++q)
        for (int i = 0; i < 2; ++i) {
          dp.push_back(o.frame_of(fl.d_dof(q, i)));
          up.push_back(o.frame_of(fl.u_dof(q, i)));
        }
      for (int e = 0; e < fl.n_elements; ++e)
        for (int k = 0; k < 3; ++k) pp.push_back(o.frame_of(fl.p_dof(e, k)));
      mesh_[l].drop = masks[l] ? constrained_positions(o, *masks[l]) : std::vector<std::uint8_t>{};
      fsigpu_mesh_desc m{fl.n_elements, fl.n_q2_nodes, 9, 2, 3, en.data(), fl.elem_solid.data(),
                         fl.node_solid.data(), dp.data(), up.data(), pp.data(),
                         mesh_[l].drop.empty() ? nullptr : mesh_[l].drop.data()};
      fsigpu_sets sets = nullptr;
      check(fsigpu_fs_sets_build(&x, &m, plan.elems_per_block, plan.elems_per_block, plan.overlap_layers, &sets));
      int n1 = 0, l1 = 0, n2 = 0, l2 = 0, nus = 0;
      fsigpu_sets_counts(sets, &n1, &l1, &n2, &l2, &nus);
      as1_ptr_[l].resize(n1 + 1);
      as1_idx_[l].resize(l1);
      as2_ptr_[l].resize(n2 + 1);
      as2_idx_[l].resize(l2);
      lumped_[l].resize(nus);
      fsigpu_sets_copy(sets, as1_ptr_[l].data(), as1_idx_[l].data(), as2_ptr_[l].data(), as2_idx_[l].data(),
                       lumped_[l].data());
      for (int b = 0; b < n1 + n2; ++b) labels_[static_cast<int>(l)].push_back(fsigpu_sets_label(sets, b));
      fsigpu_sets_destroy(sets);
      x.lumped = lumped_[l].data();
      x.as1_n = n1;
      x.as1_ptr = as1_ptr_[l].data();
      x.as1_idx = as1_idx_[l].data();
      x.as2_n = n2;
      x.as2_ptr = as2_ptr_[l].data();
      x.as2_idx = as2_idx_[l].data();
    }
    check(fsigpu_gmg_create(static_cast<int>(d.size()), d.data(), cfg.omega, cfg.pre, cfg.post, cfg.cycle, &h_),
          &labels_);
  }
  ~GpuGmg() override { fsigpu_gmg_destroy(h_); }
  int size() const override { return fsigpu_gmg_size(h_); }
  void apply(const double* r, double* z) const override { check(fsigpu_gmg_apply(h_, r, z)); }
  fsigpu_gmg handle() const { return h_; }

 private:
  fsigpu_gmg h_ = nullptr;
  std::map<size_t, std::vector<int>> as1_ptr_, as1_idx_, as2_ptr_, as2_idx_;
  std::map<int, std::vector<std::string>> labels_;  // per level: AS1 then AS2 block labels
  std::map<size_t, std::vector<double>> lumped_;
  struct MeshMaps {
    std::vector<int> en, dp, up, pp;
    std::vector<std::uint8_t> drop;
  };
  std::map<size_t, MeshMaps> mesh_;
};

// Drop-in for gmres(aop, mop, b, cfg) at driver.cpp:262-272.
GmresResult gpu_gmres(const GpuGmg& g, const std::vector<double>& frame_scale, const std::vector<double>& b,
                      const KrylovConfig& cfg) {
  fsigpu_gmres s = nullptr;
  check(fsigpu_gmres_create(g.handle(), frame_scale.data(), cfg.restart, &s));
  GmresResult out;
  out.x.resize(b.size());
  out.history.resize(static_cast<size_t>(cfg.max_iters) + 2);
  fsigpu_gmres_result r{};
  const int rc = fsigpu_gmres_solve(s, b.data(), nullptr, out.x.data(), cfg.max_iters, cfg.rel_tol, cfg.abs_tol,
                                    out.history.data(), &r);
  fsigpu_gmres_destroy(s);
  check(rc);
  out.history.resize(r.n_history);
  out.iterations = r.iterations;
  out.converged = r.converged != 0;
  out.breakdown = r.breakdown != 0;
  return out;
}

}  // namespace fsi
