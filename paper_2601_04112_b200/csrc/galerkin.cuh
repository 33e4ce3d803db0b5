// galerkin.cuh — block-structured Galerkin products (hierarchy.hpp:171-172).
#pragma once

#include "setup_kernels.cuh"
#include "sparse.cuh"

namespace lsb {

// G_{l+1} = G_l · P_l (Symbolic, bit-exact) using the panel form of P_l.
void galerkin_gp(const DevCsr& g, const DevTopo& topo, const DevInterp& ip, DevCsr& out, cudaStream_t s);
// A_{l+1} = G_{l+1}ᵀ G_{l+1} (Symbolic, bit-exact) from aggregate-pair tiles;
// rs are the level-l row sets of G_l (rows touching each aggregate).
void galerkin_gtg(const DevCsr& gn, const DevRowSets& rs, int64_t n_agg, const DevInterp& ip, const int32_t* col_agg,
                  DevCsr& out, cudaStream_t s);

}  // namespace lsb
