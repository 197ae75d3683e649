// SPDX-License-Identifier: Apache-2.0
//
// Reference-side harness (TEST INFRASTRUCTURE ONLY; never part of the product
// path). Links the UNMODIFIED reference library built by `make -C oracle ref`
// and
//   * builds the solve-phase inputs of a benchmark case exactly the way the
//     reference driver does for the first Newton iterate
//     (proj/src/driver.cpp:206-272): per-level rest-state Jacobians with
//     Dirichlet rows (assembly.cpp:220-231), J2 frames (ordering.cpp:11-13),
//     FS block sets from FsPreconditioner (precond.cpp:119-269), transfers
//     (gmg.cpp:77-136), constraint masks (driver.cpp:250-255), fine row
//     scaling (driver.cpp:150-186) and a seeded RHS (0 on constrained rows,
//     SURVEY D8);
//   * runs the reference GMRES (krylov.cpp:20-126) with the reference
//     GmgPreconditioner (gmg.cpp:178-246) and either the shipped
//     multiplicative FS smoother or the additive FS variant assembled from
//     the reference's own SchwarzSweep(..., Additive) (precond.cpp:44-57;
//     recipe SURVEY §8c);
//   * writes everything (inputs + golden outputs) to an FSIX archive that
//     the Python tests / bench read (format: see paper_1909_13201_b200/fsix.py).
//
// Usage:
//   fsi_ref_harness export <case> <out.fsix> [--seed S] [--reps R] [--no-mult]
//                          [--max-iters N] [--no-gmres] [--smoother fs|as]
//   fsi_ref_harness solve  <case> [--mode add|mult] [--reps R] [--max-iters N]
//   fsi_ref_harness blocks <out.fsix> [--seed S]     (golden dense LU blocks)
//   fsi_ref_harness time-blocks <n54> <n59> <nsolve> [--threads T] [--seed S]
//   fsi_ref_harness export3d <v3s|v3s_dd|v3|v3_dd> <out.fsix> [--no-gmres]
//                          (configs 3-4: 3D valve-like system, valve3d.inc)
// cases: cfg0 (unit square 8->16->32), sq4 (8->64, 4 levels), chan (reference
// unit_solver channel nx=4 ny_fluid=2 ny_wall=1, 2 levels), changmg (unit_gmg
// channel, ny_wall=2, 2 levels), cfg2 (bulge 16->256, 5 levels), cfg2l4 (bulge
// 16->128, 4 levels).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fsi/assembly.hpp"
#include "fsi/dense.hpp"
#include "fsi/driver.hpp"
#include "fsi/errors.hpp"
#include "fsi/gmg.hpp"
#include "fsi/krylov.hpp"
#include "fsi/ordering.hpp"
#include "fsi/precond.hpp"
#include "fsi/sparse.hpp"
#include "fsi/sparse_lu.hpp"
#ifdef FSI_ADAPTER_CHECK
#include "../../tests/cpp/gpu_solve_adapter.cpp"
#endif

using namespace fsi;

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ---------------------------------------------------------------- archive
struct Archive {
  FILE* f = nullptr;
  explicit Archive(const std::string& path) {
    f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot open " + path);
    std::fwrite("FSIX0001", 1, 8, f);
  }
  ~Archive() {
    if (f) std::fclose(f);
  }
  void put_raw(const std::string& name, const char* dt, const void* p, long long count, int esz) {
    const unsigned nl = static_cast<unsigned>(name.size());
    std::fwrite(&nl, 4, 1, f);
    std::fwrite(name.data(), 1, nl, f);
    char d[4] = {0, 0, 0, 0};
    std::memcpy(d, dt, std::min<size_t>(3, std::strlen(dt)));
    std::fwrite(d, 1, 4, f);
    std::fwrite(&count, 8, 1, f);
    if (count) std::fwrite(p, esz, count, f);
  }
  void put(const std::string& n, const std::vector<double>& v) { put_raw(n, "f8", v.data(), v.size(), 8); }
  void put(const std::string& n, const std::vector<int>& v) { put_raw(n, "i4", v.data(), v.size(), 4); }
  void put(const std::string& n, const std::vector<std::uint8_t>& v) { put_raw(n, "u1", v.data(), v.size(), 1); }
  void put_i(const std::string& n, long long x) {
    std::vector<int> v{static_cast<int>(x)};
    put(n, v);
  }
  void put_d(const std::string& n, double x) { put(n, std::vector<double>{x}); }
  void put_csr(const std::string& n, const SparseMatrix& a) {
    put_i(n + "/rows", a.rows());
    put_i(n + "/cols", a.cols());
    put(n + "/ptr", a.row_offsets());
    put(n + "/idx", a.col_indices());
    put(n + "/val", a.values());
  }
  void put_sets(const std::string& n, const std::vector<const IndexSet*>& sets) {
    std::vector<int> ptr{0}, idx;
    std::vector<std::uint8_t> labels;  // IndexSet labels, '\n'-separated
    for (auto* s : sets) {
      idx.insert(idx.end(), s->indices.begin(), s->indices.end());
      ptr.push_back(static_cast<int>(idx.size()));
      labels.insert(labels.end(), s->label.begin(), s->label.end());
      labels.push_back('\n');
    }
    put(n + "/ptr", ptr);
    put(n + "/idx", idx);
    put(n + "/labels", labels);
  }
};

// ---------------------------------------------------------------- cases
struct CaseDef {
  std::string name;
  GeometryCase geo;
  std::function<void(Mesh&)> tweak;
  int levels = 3;
  MaterialParams mat;
  std::vector<BoundaryCondition> bcs;
  double dt = 0.01;
  int epb1 = 4, epb2 = 4, overlap = 1;
  double t_eval = 0.01;
};

BoundaryCondition bc(const std::string& g, BcKind k) {
  BoundaryCondition b;
  b.group = g;
  b.kind = k;
  b.profile_peak = 0.0;
  return b;
}

std::vector<BoundaryCondition> channel_pulse_bcs(double amplitude) {
  BoundaryCondition inlet = bc("inlet", BcKind::NormalStress);
  inlet.stress_amplitude = amplitude;
  BoundaryCondition outlet = inlet;
  outlet.group = "outlet";
  outlet.stress_amplitude = -amplitude;
  return {inlet, outlet, bc("clamp_in", BcKind::DisplacementDirichlet),
          bc("clamp_out", BcKind::DisplacementDirichlet)};
}

MaterialParams cfg_material() {
  MaterialParams m;
  m.young = 1e5;
  m.poisson = 0.4;
  m.rho_s = 1000.0;
  m.rho_f = 1060.0;
  m.mu = 3.5e-3;
  return m;
}

CaseDef make_case(const std::string& name) {
  CaseDef c;
  c.name = name;
  if (name == "cfg0" || name == "sq4" || name == "sq16") {
    // unit square, bottom coarse row solid, Dirichlet
    // d and u (peak 0) on left and bottom.
    c.geo.name = "unit_square";
    c.geo.unit_n = (name == "sq16") ? 16 : 8;
    const int un = c.geo.unit_n;
    c.tweak = [un](Mesh& m) {
      for (int e = 0; e < m.n_elements(); ++e)
        if (e / un < 1) m.element_region[e] = Region::Solid;
    };
    c.levels = (name == "cfg0" || name == "sq16") ? 3 : 4;
    c.mat = cfg_material();
    c.bcs = {bc("left", BcKind::DisplacementDirichlet), bc("left", BcKind::VelocityDirichlet),
             bc("bottom", BcKind::DisplacementDirichlet), bc("bottom", BcKind::VelocityDirichlet)};
    c.dt = 0.01;
    c.t_eval = 0.01;
  } else if (name == "chan" || name == "changmg") {
    // reference unit tests' channel fixtures (tests/unit_solver.cpp:48-60,
    // tests/unit_gmg.cpp:42-50), first implicit step at the lifted rest state
    c.geo.name = "channel";
    c.geo.nx = 4;
    c.geo.ny_fluid = 2;
    c.geo.ny_wall = (name == "chan") ? 1 : 2;
    c.levels = 2;
    c.mat = MaterialParams{};
    c.bcs = channel_pulse_bcs(name == "chan" ? 15.0 : 0.1);
    c.dt = 1.0 / 32.0;
    c.t_eval = 1.0 / 32.0;
  } else if (name == "cfg2" || name == "cfg2l4") {
    // bulge, 1 coarse wall row -> 16 fine rows (D10)
    c.geo.name = "bulge";
    c.geo.length = 1.0;
    c.geo.lumen_height = 0.875;
    c.geo.wall_thickness = 0.0625;
    c.geo.nx = 16;
    c.geo.ny_fluid = 14;
    c.geo.ny_wall = 1;
    c.geo.bulge_height = 0.2;
    c.geo.bulge_width = 0.4;
    c.geo.bulge_center = 0.5;
    c.levels = (name == "cfg2") ? 5 : 4;  // cfg2l4: same case one level coarser (16 -> 128)
    c.mat = cfg_material();
    c.bcs = {bc("inlet", BcKind::DisplacementDirichlet), bc("inlet", BcKind::VelocityDirichlet),
             bc("clamp_in", BcKind::DisplacementDirichlet), bc("clamp_in", BcKind::VelocityDirichlet),
             bc("clamp_out", BcKind::DisplacementDirichlet),
             bc("clamp_out", BcKind::VelocityDirichlet)};
    c.epb1 = 4;
    c.epb2 = 16;  // D11: v,p patches 4x4 elements at levels >= 2
  } else {
    throw std::invalid_argument("unknown case " + name);
  }
  return c;
}

// build_level_stack (driver.cpp:26-57) with a caller-tweaked coarse mesh.
LevelStack make_stack(const CaseDef& c) {
  LevelStack st;
  Mesh m0 = build_case(c.geo);
  if (c.tweak) c.tweak(m0);
  st.hier.levels.push_back(std::move(m0));
  for (int l = 1; l < c.levels; ++l) refine(st.hier);
  const int levels = c.levels;
  st.spaces.reserve(levels);
  st.problems.reserve(levels);
  for (int l = 0; l < levels; ++l) st.spaces.push_back(build_layout(st.hier.levels[l], 3));
  for (int l = 0; l < levels; ++l) {
    FsiProblem p;
    p.space = &st.spaces[l];
    p.material = c.mat;
    p.kfun = KFunction{};
    p.bcs = c.bcs;
    p.scheme = TimeScheme{c.dt};
    st.problems.push_back(std::move(p));
  }
  for (int l = 0; l < levels; ++l) {
    st.assemblers.push_back(std::make_unique<Assembler>(st.problems[l]));
    st.orderings.push_back(build_orderings(st.spaces[l].layout));
  }
  for (int l = 1; l < levels; ++l) {
    st.transfers_j2.push_back(build_transfer(st.hier, l, st.spaces[l - 1], st.spaces[l],
                                             st.orderings[l - 1].j2, st.orderings[l].j2));
    st.transfers_j1.push_back(build_transfer(st.hier, l, st.spaces[l - 1], st.spaces[l],
                                             st.orderings[l - 1].j1, st.orderings[l].j1));
  }
  for (int l = 0; l < levels; ++l) st.vanka_blocks.push_back(build_vanka_blocks(st.spaces[l], c.epb1));
  return st;
}

// --smoother as: the AS (Vanka, J1) smoother (precond.cpp:99-117) instead of FS
static bool g_as = false;

// body(i) for i in [0, n), one std::thread per index (n is a few levels).
// The first exception is rethrown on the calling thread.
void parallel_for(int n, const std::function<void(int)>& body) {
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(n);
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i]() {
      try {
        body(i);
      } catch (...) {
        err[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// Additive FS smoother from the reference's own classes (SURVEY §8c recipe).
struct AdditiveFs final : LinearOperator {
  int n = 0, g1 = 0, g2 = 0, n_us = 0;
  std::unique_ptr<SchwarzSweep> as1, as2f;
  std::vector<double> lumped;
  SparseCsc csc_g2;
  AdditiveFs(const FsPreconditioner& fs, const FsPreconditioner& fs_as2) {
    n = fs.size();
    g1 = fs.group1_size();
    g2 = n - g1;
    n_us = fs.solid_velocity_size();
    std::vector<IndexSet> s1, s2;
    for (int b = 0; b < fs.as1().n_blocks(); ++b) s1.push_back(fs.as1().block_dofs(b));
    for (int b = 0; b < fs_as2.n_fluid_blocks(); ++b) s2.push_back(fs_as2.fluid_block_dofs(b));
    as1 = std::make_unique<SchwarzSweep>(fs.group1_matrix(), std::move(s1), SchwarzMode::Additive);
    as2f = std::make_unique<SchwarzSweep>(fs.group2_matrix(), std::move(s2), SchwarzMode::Additive);
    lumped = fs.lumped();
    csc_g2 = SparseCsc::from_csr(fs.group2_matrix());
  }
  // AS smoother: one additive sweep over the Vanka blocks of the J1 frame
  // (the reference's AsPreconditioner sets, precond.cpp:99-117), no split
  AdditiveFs(const AsPreconditioner& as, const SparseMatrix& frame) {
    n = frame.rows();
    g1 = n;
    g2 = 0;
    n_us = 0;
    std::vector<IndexSet> s1;
    for (int b = 0; b < as.sweep().n_blocks(); ++b) s1.push_back(as.sweep().block_dofs(b));
    as1 = std::make_unique<SchwarzSweep>(frame, std::move(s1), SchwarzMode::Additive);
    SparseMatrix empty(0, 0);
    as2f = std::make_unique<SchwarzSweep>(empty, std::vector<IndexSet>{}, SchwarzMode::Additive);
    csc_g2 = SparseCsc::from_csr(empty);
  }
  int size() const override { return n; }
  void apply(const double* r, double* z) const override {
    std::fill(z, z + n, 0.0);
    as1->apply(r, z);
    const double* r2 = r + g1;
    double* z2 = z + g1;
    std::vector<double> res(r2, r2 + g2), t(g2);
    for (int i = 0; i < n_us; ++i) {
      const double d = r2[i] / lumped[i];
      z2[i] = d;
      if (d == 0.0) continue;
      for (int k = csc_g2.col_offsets[i]; k < csc_g2.col_offsets[i + 1]; ++k)
        res[csc_g2.row_indices[k]] -= csc_g2.values[k] * d;
    }
    as2f->apply(res.data(), t.data());
    for (int i = 0; i < g2; ++i) z2[i] += t[i];
  }
};

struct Problem {
  CaseDef def;
  LevelStack st;
  int top = 0, n = 0;
  std::vector<SparseMatrix> frame;
  std::vector<std::vector<Constraint>> cs;
  std::vector<ConstraintMasks> cmask;
  std::vector<std::unique_ptr<FsPreconditioner>> fs, fs_as2;  // as2 sets from epb2 instance
  std::vector<std::unique_ptr<AsPreconditioner>> as_mult;    // --smoother as
  std::vector<std::unique_ptr<AdditiveFs>> fs_add;
  std::vector<GmgLevel> levels_mult, levels_add;
  std::unique_ptr<GmgPreconditioner> gmg_mult, gmg_add;
  SparseMatrix a_scaled;
  std::vector<double> frame_scale, b;
  double setup_assembly_s = 0, setup_fs_s = 0, setup_coarse_s = 0;
};

std::unique_ptr<Problem> build_problem(const std::string& name, unsigned long long seed, bool want_mult) {
  auto P = std::make_unique<Problem>();
  P->def = make_case(name);
  double t0 = now_s();
  P->st = make_stack(P->def);
  LevelStack& st = P->st;
  const int L = st.n_levels();
  const int top = L - 1;
  P->top = top;
  const double t = P->def.t_eval;

  // state: rest state lifted (first Newton iterate)
  std::vector<double> x_fine = rest_state(st.spaces[top], st.problems[top].material);
  std::vector<std::vector<double>> xo(L), xl(L);
  xo[top] = x_fine;
  for (int l = top - 1; l >= 0; --l)
    xo[l] = restrict_state(st.hier, l + 1, st.spaces[l], st.spaces[l + 1], xo[l + 1]);
  std::vector<StabilizationState> stab(L);
  for (int l = 0; l <= top; ++l) stab[l] = compute_stabilization(st.problems[l], xo[l]);
  P->cs.resize(L);
  P->cmask.resize(L);
  for (int l = 0; l <= top; ++l) {
    P->cs[l] = build_constraints(st.problems[l], t);
    P->cmask[l].rows.assign(st.spaces[l].layout.n_dofs, 0);
    P->cmask[l].dofs.assign(st.spaces[l].layout.n_dofs, 0);
    for (const auto& c : P->cs[l]) {
      P->cmask[l].rows[c.row] = 1;
      P->cmask[l].dofs[c.dof] = 1;
    }
  }
  lift_constraints(P->cs[top], x_fine);
  xl[top] = x_fine;
  for (int l = top - 1; l >= 0; --l)
    xl[l] = restrict_state(st.hier, l + 1, st.spaces[l], st.spaces[l + 1], xl[l + 1]);

  // the levels are independent objects of the reference (no shared mutable
  // state), so they are assembled on one host thread each
  P->frame.resize(L);
  SparseMatrix jac_top;
  parallel_for(L, [&](int l) {
    st.assemblers[l]->assemble(xl[l], xo[l], xo[l], stab[l], t, true);
    SparseMatrix jl = st.assemblers[l]->jacobian();
    std::vector<double> rl = st.assemblers[l]->residual();
    apply_dirichlet(jl, rl, P->cs[l], xl[l]);
    P->frame[l] = (g_as ? st.orderings[l].j1 : st.orderings[l].j2).apply(jl);
    if (l == top) jac_top = std::move(jl);
  });
  P->setup_assembly_s = now_s() - t0;

  t0 = now_s();
  P->fs.resize(L);
  P->fs_as2.resize(L);
  P->fs_add.resize(L);
  P->as_mult.resize(L);
  for (int l = 1; l <= top && g_as; ++l) {
    P->as_mult[l] = std::make_unique<AsPreconditioner>(P->frame[l], st.orderings[l].j1, st.vanka_blocks[l],
                                                       &P->cmask[l]);
    P->fs_add[l] = std::make_unique<AdditiveFs>(*P->as_mult[l], P->frame[l]);
  }
  // FS instances (level x {epb1, epb2}) built on one host thread each
  if (!g_as) {
    const bool two = P->def.epb2 != P->def.epb1;
    parallel_for(2 * L, [&](int task) {
      const int l = task / 2;
      if (l == 0 || (task % 2 == 1 && !two)) return;
      const int epb = task % 2 == 0 ? P->def.epb1 : P->def.epb2;
      auto f = std::make_unique<FsPreconditioner>(P->frame[l], st.orderings[l].j2, st.spaces[l],
                                                  FieldSplitPlan{epb, P->def.overlap}, &P->cmask[l]);
      (task % 2 == 0 ? P->fs[l] : P->fs_as2[l]) = std::move(f);
    });
    for (int l = 1; l <= top; ++l)
      P->fs_add[l] = std::make_unique<AdditiveFs>(*P->fs[l], two ? *P->fs_as2[l] : *P->fs[l]);
  }
  P->setup_fs_s = now_s() - t0;

  auto fill_levels = [&](std::vector<GmgLevel>& lv, bool additive) {
    lv.resize(L);
    for (int l = 0; l <= top; ++l) {
      GmgLevel& g = lv[l];
      g.a = &P->frame[l];
      g.smoother = (l == 0) ? nullptr
                   : additive ? static_cast<const LinearOperator*>(P->fs_add[l].get())
                   : g_as     ? static_cast<const LinearOperator*>(P->as_mult[l].get())
                              : static_cast<const LinearOperator*>(P->fs[l].get());
      if (l > 0) {
        g.p = (g_as ? st.transfers_j1 : st.transfers_j2)[l - 1].p;
        g.r = (g_as ? st.transfers_j1 : st.transfers_j2)[l - 1].r;
      }
      const OrderingPlan& plan = g_as ? st.orderings[l].j1 : st.orderings[l].j2;
      g.constrained_rows.assign(st.spaces[l].layout.n_dofs, 0);
      g.constrained_cols.assign(st.spaces[l].layout.n_dofs, 0);
      for (const auto& c : P->cs[l]) {
        g.constrained_rows[plan.row_to[c.row]] = 1;
        g.constrained_cols[plan.col_to[c.dof]] = 1;
      }
    }
  };
  CycleConfig cyc{'v', 1, 1, 0.7};
  t0 = now_s();
  fill_levels(P->levels_add, true);
  P->gmg_add = std::make_unique<GmgPreconditioner>(P->levels_add, cyc);
  P->setup_coarse_s = now_s() - t0;
  if (want_mult) {
    fill_levels(P->levels_mult, false);
    P->gmg_mult = std::make_unique<GmgPreconditioner>(P->levels_mult, cyc);
  }

  // fine row scaling (driver.cpp:150-186) and the frame RHS
  const int n = st.spaces[top].layout.n_dofs;
  P->n = n;
  std::vector<double> row_scale(n, 1.0);
  {
    const auto& vals = jac_top.values();
    const auto& off = jac_top.row_offsets();
    for (int i = 0; i < n; ++i) {
      double mx = 0.0;
      for (int k = off[i]; k < off[i + 1]; ++k) mx = std::max(mx, std::abs(vals[k]));
      if (mx > 0.0) row_scale[i] = 1.0 / mx;
    }
  }
  SparseMatrix jac_scaled = jac_top;
  {
    auto& vals = jac_scaled.values();
    const auto& off = jac_scaled.row_offsets();
    for (int i = 0; i < n; ++i)
      for (int k = off[i]; k < off[i + 1]; ++k) vals[k] *= row_scale[i];
  }
  const OrderingPlan& plan_top = g_as ? st.orderings[top].j1 : st.orderings[top].j2;
  P->a_scaled = plan_top.apply(jac_scaled);
  P->frame_scale.resize(n);
  for (int i = 0; i < n; ++i) P->frame_scale[i] = row_scale[plan_top.row_from[i]];
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  P->b.assign(n, 0.0);
  const auto& crow = P->levels_add[top].constrained_rows;
  for (int i = 0; i < n; ++i) {
    const double v = U(rng);
    P->b[i] = crow[i] ? 0.0 : v;
  }
  return P;
}

struct SolveOut {
  GmresResult res;
  long long m_applies = 0;
  double seconds = 0;
  double true_res = 0;
};

SolveOut run_gmres(const Problem& P, bool additive, const KrylovConfig& kc) {
  const int n = P.n;
  const GmgPreconditioner& g = additive ? *P.gmg_add : *P.gmg_mult;
  SolveOut out;
  CsrOperator aop(P.a_scaled);
  long long* cnt = &out.m_applies;
  FunctionOperator mop(n, [&, cnt](const double* r, double* z) {
    ++*cnt;
    std::vector<double> unscaled(n);
    for (int i = 0; i < n; ++i) unscaled[i] = r[i] / P.frame_scale[i];
    g.apply(unscaled.data(), z);
  });
  const double t0 = now_s();
  out.res = gmres(aop, mop, P.b, kc);
  out.seconds = now_s() - t0;
  auto ax = P.a_scaled.multiply(out.res.x);
  double s = 0;
  for (int i = 0; i < n; ++i) s += (P.b[i] - ax[i]) * (P.b[i] - ax[i]);
  out.true_res = std::sqrt(s);
  return out;
}

struct Args {
  std::vector<std::string> pos;
  unsigned long long seed = 20240901ull;
  int reps = 1, max_iters = 2000, threads = 1, block_stride = 1;
  double rtol = 1e-10;
  bool no_mult = false, no_gmres = false;
  std::string mode = "add";
};

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string s = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + s);
      return argv[++i];
    };
    if (s == "--seed") a.seed = std::stoull(next());
    else if (s == "--reps") a.reps = std::stoi(next());
    else if (s == "--max-iters") a.max_iters = std::stoi(next());
    else if (s == "--threads") a.threads = std::stoi(next());
    else if (s == "--rtol") a.rtol = std::stod(next());
    else if (s == "--block-stride") a.block_stride = std::stoi(next());
    else if (s == "--smoother") g_as = (next() == "as");
    else if (s == "--mode") a.mode = next();
    else if (s == "--no-mult") a.no_mult = true;
    else if (s == "--no-gmres") a.no_gmres = true;
    else a.pos.push_back(s);
  }
  return a;
}

void put_solve(Archive& ar, const std::string& pre, const SolveOut& s) {
  ar.put(pre + "/x", s.res.x);
  ar.put(pre + "/history", s.res.history);
  ar.put_i(pre + "/iterations", s.res.iterations);
  ar.put_i(pre + "/converged", s.res.converged ? 1 : 0);
  ar.put_i(pre + "/m_applies", s.m_applies);
  ar.put_d(pre + "/seconds", s.seconds);
  ar.put_d(pre + "/true_residual", s.true_res);
}

std::vector<double> seeded(int n, std::mt19937_64& rng) {
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> v(n);
  for (auto& x : v) x = U(rng);
  return v;
}

// The mesh-side inputs of the FS / Vanka block construction
// (FsPreconditioner ctor, precond.cpp:119-269; build_vanka_blocks +
// AsPreconditioner, ordering.cpp:77-115, precond.cpp:99-117) in the
// solver's frame: element -> Q2 nodes, the region flags, the frame
// positions of every d, u and p dof (OrderingPlan::frame_of) and the
// dropped positions (constrained_positions, precond.cpp:90-97), so the GPU
// can build the block sets itself (fsigpu_fs_sets_build).
void put_mesh(Archive& ar, const std::string& pre, const Problem& P, int l) {
  const Space& sp = P.st.spaces[l];
  const FieldLayout& fl = sp.layout;
  const OrderingPlan& plan = g_as ? P.st.orderings[l].j1 : P.st.orderings[l].j2;
  std::vector<int> en, dpos, upos, ppos;
  for (int e = 0; e < fl.n_elements; ++e)
    for (int a = 0; a < 9; ++a) en.push_back(sp.dofmap.element_nodes[e][a]);
  for (int q = 0; q < fl.n_q2_nodes; ++q)
    for (int i = 0; i < 2; ++i) {
      dpos.push_back(plan.frame_of(fl.d_dof(q, i)));
      upos.push_back(plan.frame_of(fl.u_dof(q, i)));
    }
  for (int e = 0; e < fl.n_elements; ++e)
    for (int m = 0; m < 3; ++m) ppos.push_back(plan.frame_of(fl.p_dof(e, m)));
  ar.put(pre + "/element_nodes", en);
  ar.put(pre + "/elem_solid", fl.elem_solid);
  ar.put(pre + "/node_solid", fl.node_solid);
  ar.put(pre + "/d_pos", dpos);
  ar.put(pre + "/u_pos", upos);
  ar.put(pre + "/p_pos", ppos);
  ar.put(pre + "/drop", constrained_positions(plan, P.cmask[l]));
  ar.put_i(pre + "/epb_as1", P.def.epb1);
  ar.put_i(pre + "/epb_as2", P.def.epb2);
  ar.put_i(pre + "/overlap", P.def.overlap);
}

int cmd_export(const Args& a) {
  if (a.pos.size() < 3) throw std::invalid_argument("export <case> <out>");
  const std::string name = a.pos[1];
  auto P = build_problem(name, a.seed, !a.no_mult);
  Archive ar(a.pos[2]);
  const int L = P->st.n_levels();
  ar.put_i("levels", L);
  ar.put_i("seed", static_cast<long long>(a.seed % 2147483647ull));
  for (int l = 0; l < L; ++l) {
    const std::string p = "L" + std::to_string(l);
    put_mesh(ar, p + "/mesh", *P, l);
    ar.put_csr(p + "/A", P->frame[l]);
    ar.put(p + "/row_mask", P->levels_add[l].constrained_rows);
    ar.put(p + "/col_mask", P->levels_add[l].constrained_cols);
    if (l > 0) {
      ar.put_csr(p + "/P", P->levels_add[l].p);
      ar.put_csr(p + "/R", P->levels_add[l].r);
      const AdditiveFs& f = *P->fs_add[l];
      ar.put_i(p + "/g1", f.g1);
      ar.put_i(p + "/n_us", f.n_us);
      ar.put(p + "/lumped", f.lumped);
      std::vector<const IndexSet*> s1, s2;
      for (int b = 0; b < f.as1->n_blocks(); ++b) s1.push_back(&f.as1->block_dofs(b));
      for (int b = 0; b < f.as2f->n_blocks(); ++b) s2.push_back(&f.as2f->block_dofs(b));
      ar.put_sets(p + "/as1", s1);
      ar.put_sets(p + "/as2", s2);
    }
  }
  ar.put("frame_scale", P->frame_scale);
  ar.put("b", P->b);
  ar.put_d("setup/assembly_s", P->setup_assembly_s);
  ar.put_d("setup/fs_s", P->setup_fs_s);
  ar.put_d("setup/coarse_s", P->setup_coarse_s);

  // golden intermediate outputs on the fine level
  std::mt19937_64 rng(a.seed + 17);
  const int top = P->top;
  const int n = P->n;
  {
    auto r = seeded(n, rng);
    std::vector<double> z(n);
    P->fs_add[top]->apply(r.data(), z.data());
    ar.put("golden/fs_r", r);
    ar.put("golden/fs_z_add", z);
    if (P->fs[top]) {
      P->fs[top]->apply(r.data(), z.data());
      ar.put("golden/fs_z_mult", z);
    } else if (P->as_mult[top]) {
      P->as_mult[top]->apply(r.data(), z.data());
      ar.put("golden/fs_z_mult", z);
    }
    // per-block dense solves (AS1 then AS2 blocks of the fine level)
    const AdditiveFs& f = *P->fs_add[top];
    std::vector<double> rhs, xs;
    std::vector<int> ids;  // sampled block ids (AS1 then AS2 numbering)
    const int stride = std::max(1, a.block_stride);
    for (int b = 0; b < f.as1->n_blocks(); b += stride) {
      ids.push_back(b);
      const IndexSet& s = f.as1->block_dofs(b);
      auto lu = factor_principal_block(g_as ? P->frame[top] : P->fs[top]->group1_matrix(), s);
      auto bb = seeded(s.size(), rng);
      auto xx = lu.solve(bb);
      rhs.insert(rhs.end(), bb.begin(), bb.end());
      xs.insert(xs.end(), xx.begin(), xx.end());
    }
    for (int b = 0; b < f.as2f->n_blocks(); b += stride) {
      ids.push_back(f.as1->n_blocks() + b);
      const IndexSet& s = f.as2f->block_dofs(b);
      auto lu = factor_principal_block(P->fs[top]->group2_matrix(), s);  // FS only (AS has no AS2)
      auto bb = seeded(s.size(), rng);
      auto xx = lu.solve(bb);
      rhs.insert(rhs.end(), bb.begin(), bb.end());
      xs.insert(xs.end(), xx.begin(), xx.end());
    }
    ar.put("golden/block_ids", ids);
    ar.put("golden/block_rhs", rhs);
    ar.put("golden/block_x", xs);
    // one V-cycle of the additive GMG
    auto rv = seeded(n, rng);
    std::vector<double> zv(n);
    P->gmg_add->apply(rv.data(), zv.data());
    ar.put("golden/vcycle_r", rv);
    ar.put("golden/vcycle_z_add", zv);
    // one fine-level SpMV and the coarse solve
    auto xv = seeded(n, rng);
    ar.put("golden/spmv_x", xv);
    ar.put("golden/spmv_y", P->frame[top].multiply(xv));
    const int n0 = P->frame[0].rows();
    auto b0 = seeded(n0, rng);
    SparseLu lu0(P->frame[0], true, "gmg-coarse");
    ar.put("golden/coarse_b", b0);
    ar.put("golden/coarse_x", lu0.solve(b0));
  }

  if (!a.no_gmres) {
    KrylovConfig kc;
    kc.restart = 30;
    kc.rel_tol = a.rtol;
    kc.abs_tol = 1e-300;
    kc.max_iters = a.max_iters;
    ar.put_d("gmres/rel_tol", a.rtol);
    auto sa = run_gmres(*P, true, kc);
    put_solve(ar, "gmres_add", sa);
    // the reference's default KrylovConfig (restart 60, krylov.hpp:42-47),
    // the configuration the drop-in sees from the driver (config.hpp:61)
    if (a.max_iters >= 500) {
      const KrylovConfig kd{};
      auto sd = run_gmres(*P, true, kd);
      put_solve(ar, "gmres_default", sd);
      std::printf("%s additive default KrylovConfig (restart %d): its=%d conv=%d relres=%.3e\n", name.c_str(),
                  kd.restart, sd.res.iterations, (int)sd.res.converged, sd.true_res / sd.res.history.front());
    }
    std::printf("%s additive %s: its=%d conv=%d M=%lld %.3fs relres=%.3e\n", name.c_str(), g_as ? "AS" : "FS",
                sa.res.iterations, (int)sa.res.converged, sa.m_applies, sa.seconds,
                sa.true_res / sa.res.history.front());
    if (!a.no_mult) {
      auto sm = run_gmres(*P, false, kc);
      put_solve(ar, "gmres_mult", sm);
      std::printf("%s multiplicative %s: its=%d conv=%d M=%lld %.3fs relres=%.3e\n", name.c_str(), g_as ? "AS" : "FS",
                  sm.res.iterations, (int)sm.res.converged, sm.m_applies, sm.seconds,
                  sm.true_res / sm.res.history.front());
    }
  }
  std::printf("%s: levels=%d n=%d nnz=%lld setup asm=%.2fs fs=%.2fs coarse=%.2fs\n", name.c_str(), L,
              P->n, (long long)P->frame[top].nnz(), P->setup_assembly_s, P->setup_fs_s,
              P->setup_coarse_s);
  return 0;
}

// Reference-arm timing: one GMRES solve per rep, JSON on stdout.
int cmd_solve(const Args& a) {
  if (a.pos.size() < 2) throw std::invalid_argument("solve <case>");
  const bool additive = a.mode != "mult";
  auto P = build_problem(a.pos[1], a.seed, !additive);
  KrylovConfig kc;
  kc.restart = 30;
  kc.rel_tol = a.rtol;
  kc.abs_tol = 1e-300;
  kc.max_iters = a.max_iters;
  std::printf("{\"case\": \"%s\", \"mode\": \"%s\", \"n\": %d, \"setup_s\": %.6f, \"solves\": [",
              a.pos[1].c_str(), additive ? "add" : "mult", P->n,
              P->setup_assembly_s + P->setup_fs_s + P->setup_coarse_s);
  for (int r = 0; r < a.reps; ++r) {
    auto s = run_gmres(*P, additive, kc);
    std::printf("%s{\"iterations\": %d, \"m_applies\": %lld, \"seconds\": %.6f, \"relres\": %.6e, "
                "\"converged\": %d}",
                r ? ", " : "", s.res.iterations, s.m_applies, s.seconds,
                s.true_res / s.res.history.front(), (int)s.res.converged);
    std::fflush(stdout);
  }
  std::printf("]}\n");
  return 0;
}

// Golden dense blocks: config-1 style (diagonally dominant) plus random
// non-dominant blocks that force row swaps, and a singular block.
int cmd_blocks(const Args& a) {
  if (a.pos.size() < 2) throw std::invalid_argument("blocks <out>");
  std::mt19937_64 rng(a.seed);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  Archive ar(a.pos[1]);
  std::vector<int> ptr{0}, sizes, kinds, swaps;
  std::vector<double> mats, lus, rhs, xs;
  std::vector<int> pivs;
  struct Spec { int m; int kind; };  // kind 0: dominant, 1: random (pivoting), 2: graded
  std::vector<Spec> specs;
  for (int i = 0; i < 6; ++i) specs.push_back({54, 0});
  for (int i = 0; i < 6; ++i) specs.push_back({59, 0});
  for (int m : {1, 2, 3, 7, 31, 32, 33, 44, 63, 64, 65, 97, 128, 162}) specs.push_back({m, 1});
  for (int m : {40, 108, 162}) specs.push_back({m, 2});
  for (const auto& sp : specs) {
    const int m = sp.m;
    DenseMatrix d(m, m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) d(i, j) = U(rng);
    if (sp.kind == 0) {
      for (int i = 0; i < m; ++i) {
        double s = 0;
        for (int j = 0; j < m; ++j) s += std::abs(d(i, j));
        d(i, i) += s;
      }
    } else if (sp.kind == 2) {
      // wide row scales like the J2 blocks (1e-6 .. 1e5)
      for (int i = 0; i < m; ++i) {
        const double sc = std::pow(10.0, -6.0 + 11.0 * (i % 7) / 6.0);
        for (int j = 0; j < m; ++j) d(i, j) *= sc;
        d(i, i) += 2.0 * sc * m;
      }
    }
    DenseFactorization lu(d, "golden");
    std::vector<double> b(m);
    for (auto& v : b) v = U(rng);
    auto x = lu.solve(b);
    mats.insert(mats.end(), d.a.begin(), d.a.end());
    rhs.insert(rhs.end(), b.begin(), b.end());
    xs.insert(xs.end(), x.begin(), x.end());
    sizes.push_back(m);
    kinds.push_back(sp.kind);
  }
  ar.put("sizes", sizes);
  ar.put("kinds", kinds);
  ar.put("a", mats);
  ar.put("b", rhs);
  ar.put("x", xs);
  // singular example (tests/unit_linalg.cpp:244-247)
  DenseMatrix s(2, 2);
  s(0, 0) = s(0, 1) = s(1, 0) = s(1, 1) = 1.0;
  int singular = 0;
  std::string msg;
  try {
    DenseFactorization f(s, "wall-block");
  } catch (const SingularBlockError& e) {
    singular = 1;
    msg = e.what();
  }
  ar.put_i("singular_thrown", singular);
  std::vector<std::uint8_t> mb(msg.begin(), msg.end());
  ar.put("singular_msg", mb);
  std::printf("blocks: %zu golden blocks, singular='%s'\n", sizes.size(), msg.c_str());
  return 0;
}

// CPU baseline for config 1: DenseFactorization ctor + solves, threaded.
int cmd_time_blocks(const Args& a) {
  if (a.pos.size() < 4) throw std::invalid_argument("time-blocks <n54> <n59> <nsolve>");
  const long n54 = std::stol(a.pos[1]), n59 = std::stol(a.pos[2]);
  const int nsolve = std::stoi(a.pos[3]);
  const long nb = n54 + n59;
  const int T = std::max(1, a.threads);
  std::vector<double> lu_s(T, 0), sv_s(T, 0);
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    th.emplace_back([&, t]() {
      std::mt19937_64 rng(a.seed + 1000003ull * t);
      std::uniform_real_distribution<double> U(-1.0, 1.0);
      std::vector<DenseFactorization> fs;
      std::vector<std::vector<double>> rhs;
      double tl = 0;
      for (long b = t; b < nb; b += T) {
        const int m = (b < n54) ? 54 : 59;
        DenseMatrix d(m, m);
        for (int i = 0; i < m; ++i) {
          double s = 0;
          for (int j = 0; j < m; ++j) {
            d(i, j) = U(rng);
            s += std::abs(d(i, j));
          }
          d(i, i) += s;
        }
        const double t0 = now_s();
        fs.emplace_back(d, "b");
        tl += now_s() - t0;
        std::vector<double> r(m);
        for (auto& v : r) v = U(rng);
        rhs.push_back(std::move(r));
      }
      std::vector<double> x(64);
      const double t1 = now_s();
      for (int s = 0; s < nsolve; ++s)
        for (size_t k = 0; k < fs.size(); ++k) fs[k].solve(rhs[k].data(), x.data());
      sv_s[t] = now_s() - t1;
      lu_s[t] = tl;
    });
  }
  for (auto& x : th) x.join();
  double lu = 0, sv = 0;
  for (int t = 0; t < T; ++t) {
    lu = std::max(lu, lu_s[t]);
    sv = std::max(sv, sv_s[t]);
  }
  std::printf("{\"blocks\": %ld, \"threads\": %d, \"lu_s\": %.6f, \"solve_s_per_pass\": %.6f}\n", nb, T,
              lu, nsolve ? sv / nsolve : 0.0);
  return 0;
}

#include "valve3d.inc"

#ifdef FSI_ADAPTER_CHECK
// The drop-in adapter (tests/cpp/gpu_solve_adapter.cpp) driven like the
// reference driver's solve block (driver.cpp:242-272): GpuGmg from the
// GmgLevels + per-level FsPreconditioners, gpu_gmres with the reference's
// default KrylovConfig, against the reference's own gmres on the additive
// FS hierarchy with the same config. JSON on stdout.
int cmd_gpu_adapter(const Args& a) {
  if (a.pos.size() < 2) throw std::invalid_argument("gpu-adapter <case>");
  auto P = build_problem(a.pos[1], a.seed, false);
  const int L = P->st.n_levels();
  std::vector<const FsPreconditioner*> fs(L, nullptr);
  for (int l = 1; l < L; ++l) fs[l] = P->fs[l].get();
  const CycleConfig cyc{'v', 1, 1, 0.7};
  GpuGmg gpu(P->levels_add, fs, cyc);
  // one V-cycle through the LinearOperator interface
  std::mt19937_64 rng(a.seed + 5);
  auto r = seeded(P->n, rng);
  std::vector<double> zg(P->n), zr(P->n);
  gpu.apply(r.data(), zg.data());
  P->gmg_add->apply(r.data(), zr.data());
  double num = 0, den = 0;
  for (int i = 0; i < P->n; ++i) {
    num += (zg[i] - zr[i]) * (zg[i] - zr[i]);
    den += zr[i] * zr[i];
  }
  const KrylovConfig kc{};
  auto ref = run_gmres(*P, true, kc);
  const GmresResult g = gpu_gmres(gpu, P->frame_scale, P->b, kc);
  // the same drop-in without any reference FsPreconditioner: block sets and
  // lumped mass built on the GPU from the Space / J2 plan / masks
  std::vector<const Space*> sps;
  std::vector<const OrderingPlan*> plans;
  std::vector<const ConstraintMasks*> cms;
  for (int l = 0; l < L; ++l) {
    sps.push_back(&P->st.spaces[l]);
    plans.push_back(&P->st.orderings[l].j2);
    cms.push_back(&P->cmask[l]);
  }
  GpuGmg gpu_mesh(P->levels_add, sps, plans, cms, FieldSplitPlan{P->def.epb1, P->def.overlap}, cyc);
  const GmresResult gm = gpu_gmres(gpu_mesh, P->frame_scale, P->b, kc);
  std::vector<double> zm(P->n);
  gpu_mesh.apply(r.data(), zm.data());
  bool same = gm.iterations == g.iterations && gm.x == g.x && zm == zg;
  auto ax = P->a_scaled.multiply(g.x);
  double s2 = 0;
  for (int i = 0; i < P->n; ++i) s2 += (P->b[i] - ax[i]) * (P->b[i] - ax[i]);
  // a singular FS block surfaces as SingularBlockError with the reference label
  std::string label, expected;
  {
    std::vector<GmgLevel> bad = P->levels_add;
    SparseMatrix broken = P->frame[L - 1];
    const IndexSet& s0 = P->fs[L - 1]->fluid_block_dofs(3);
    const int row = P->fs[L - 1]->group1_size() + s0.indices[0];
    // the lowest AS2 block holding that dof is the one reported
    for (int b = 0; b < P->fs[L - 1]->n_fluid_blocks() && expected.empty(); ++b)
      if (P->fs[L - 1]->fluid_block_dofs(b).contains(s0.indices[0])) expected = P->fs[L - 1]->fluid_block_dofs(b).label;
    for (int k = broken.row_offsets()[row]; k < broken.row_offsets()[row + 1]; ++k) broken.values()[k] = 0.0;
    bad[L - 1].a = &broken;
    try {
      GpuGmg g2(bad, fs, cyc);
    } catch (const SingularBlockError& e) {
      label = e.label();
    }
  }
  std::printf("{\"case\": \"%s\", \"restart\": %d, \"vcycle_rel\": %.3e, \"ref_iterations\": %d, "
              "\"ref_converged\": %d, \"ref_relres\": %.6e, \"gpu_iterations\": %d, \"gpu_converged\": %d, "
              "\"gpu_relres\": %.6e, \"singular_label\": \"%s\", \"expected_label\": \"%s\", "
              "\"device_sets_identical\": %d}\n",
              a.pos[1].c_str(), kc.restart, std::sqrt(num / den), ref.res.iterations, (int)ref.res.converged,
              ref.true_res / ref.res.history.front(), g.iterations, (int)g.converged,
              std::sqrt(s2) / g.history.front(), label.c_str(), expected.c_str(), (int)same);
  return 0;
}
#endif

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse(argc, argv);
    if (a.pos.empty()) {
      std::fprintf(stderr, "usage: fsi_ref_harness export|solve|blocks|time-blocks ...\n");
      return 2;
    }
    const std::string& c = a.pos[0];
    if (c == "export") return cmd_export(a);
    if (c == "solve") return cmd_solve(a);
    if (c == "blocks") return cmd_blocks(a);
    if (c == "time-blocks") return cmd_time_blocks(a);
    if (c == "export3d") return cmd_export3d(a);
#ifdef FSI_ADAPTER_CHECK
    if (c == "gpu-adapter") return cmd_gpu_adapter(a);
#endif
    std::fprintf(stderr, "unknown command %s\n", c.c_str());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
