// Nyström PCG driver on device (solvers.cpp:40-148): batched over S
// independent right-hand sides that share one pass over A per iteration.
#pragma once

#include <string>
#include <vector>

#include "ops.cuh"

namespace npcg {

struct PcgOptions {
  double eta = 1e-10;
  i64 max_iter = 500;
  bool relative = false;
  bool record_iterates = false;
};

struct PcgColumnReport {
  i64 iterations = 0;
  i64 matvec_count = 0;
  bool converged = false;
  int status = 0;  // 0 ok / max_iter, 1 breakdown, 2 non-finite residual, 3 non-finite initial residual
  double eta_used = 0.0;
  std::vector<double> history;
};

struct PcgResult {
  std::vector<PcgColumnReport> cols;
  double wall_time = 0.0;
  bool diverged = false;
  std::string message;
};

/// Device record of the iterates (record_iterates, solvers.hpp:24): layout
/// [t][s][n] for t < cap, zero where a column did not run; grown by doubling
/// as the loop advances (not sized for max_iter up front).
struct IterateRec {
  DBuf<double> buf;
  i64 cap = 0;  // iterations the buffer holds
};

/// Columns with their own shift: column s solves (A + mu[s] I) x = b_s with pre[s]
/// (all built from one factorisation). One pass over A per iteration serves
/// every column, so a cold-start regularisation path batches several mu.
struct PcgMuCols {
  std::vector<double> mu;
  std::vector<Pre*> pre;
};
/// Whether pcg_solve takes per-column shifts for this operator and column count.
bool pcg_mu_batch_eligible(Ctx& ctx, Op& op, i64 S);

/// Solves (A + mu I) X = B column by column with P^{-1} from `pre`
/// (nullptr = identity, i.e. cg() on A + mu I). B, X0, X are device n x S
/// (X0 nullable = 0). `iterates` (nullable): filled with x_0 .. x_t.
PcgResult pcg_solve(Ctx& ctx, Op& op, Pre* pre, double mu, i64 S, const double* B, i64 ldb, const double* X0,
                    i64 ldx0, const PcgOptions& opt, double* X, i64 ldx, IterateRec* iterates,
                    const char* context = "nystrom_pcg", const PcgMuCols* cols = nullptr);

struct BlockPcgResult {
  i64 iterations = 0;
  i64 fallback_count = 0;
  std::vector<i64> deflated;
  std::vector<bool> converged;
  std::vector<std::vector<double>> history;
  double eta_used = 0.0;
  double wall_time = 0.0;
};

/// block_nystrom_pcg (solvers.cpp:150-279) on device; B, X device n x s (s <= 8).
BlockPcgResult block_pcg_solve(Ctx& ctx, Op& op, Pre* pre, double mu, i64 s, const double* B, i64 ldb,
                               const PcgOptions& opt, double* X, i64 ldx);

}  // namespace npcg
