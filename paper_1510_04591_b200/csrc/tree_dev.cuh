// Device view of an HSS tree (hsseig_tree) shared by the randomized (hss_build.cu) and
// the SRRSC (srrsc.cu) constructions.
#pragma once
#include "common.cuh"

namespace hsseig {

constexpr double kTol3z = 1.0536712127723509e-08;  // sqrt(dlamch('E')) = sqrt(2^-53)
constexpr double kFlagTol = 1e-12;                  // hss.py:117

struct TreeDev {
  int32_t k, n_leaves, depth, w, ws, pmax, mmax;
  const int32_t *lo, *hi, *left, *right, *lnodes;
  int32_t *rU, *rV, *rsel, *csel, *rloc, *cloc, *flags;
  double *U, *V, *Vt, *B, *D, *rres, *cres, *M, *psel, *tsel, *ycomp, *zcomp;
  int32_t dld;
};

static inline TreeDev to_dev(const hsseig_tree* t) {
  TreeDev d;
  d.k = t->k; d.n_leaves = t->n_leaves; d.depth = t->depth; d.w = t->w; d.ws = t->ws;
  d.pmax = t->pmax; d.mmax = t->mmax;
  d.lo = t->lo; d.hi = t->hi; d.left = t->left; d.right = t->right; d.lnodes = t->level_nodes;
  d.rU = t->rU; d.rV = t->rV; d.rsel = t->rsel; d.csel = t->csel; d.rloc = t->rloc;
  d.cloc = t->cloc; d.flags = t->flags;
  d.U = t->U; d.V = t->V; d.Vt = t->Vt; d.dld = t->dld; d.B = t->B; d.D = t->D; d.rres = t->rres; d.cres = t->cres;
  d.M = t->M; d.psel = t->psel; d.tsel = t->tsel; d.ycomp = t->ycomp; d.zcomp = t->zcomp;
  return d;
}

__device__ __forceinline__ size_t slot_pw(const TreeDev& T, int node) {
  return (size_t)node * T.pmax * T.ws;
}
__device__ __forceinline__ size_t slot_ww(const TreeDev& T, int node) {
  return (size_t)node * T.ws * T.ws;
}

// B slots of the children of the nodes [j0, j0 + cnt) of one level (genB_kernel)
int launch_genB(const CauchyGen& g, const TreeDev& T, int level, int j0, int cnt, cudaStream_t s);

}  // namespace hsseig
