// ertinv_gnw.hpp -- the reference's own Woodbury-MINRES types backed by libgnw (the drop-in).
//
// Built INSIDE an ertinv (reference) tree: paper_2209_02815_b200/dropin/ertinv_gnw.cpp compiles
// against the reference's headers and defines, in place of proj/src/inversion.cpp's,
//     Vector SaddleOperator::apply(std::span<const double>) const            (inversion.hpp:25)
//     Vector WoodburyPreconditioner::apply(std::span<const double>) const    (inversion.hpp:38)
//     WoodburyPreconditioner build_woodbury_preconditioner(q_diag_inv, amg, J, beta, timings*)
//                                                                            (inversion.hpp:47-50)
// so callers written against the reference -- SaddleOperator{&Q, &D, &J, beta}, a default-
// constructed WoodburyPreconditioner with assigned fields, pc.capacitance_chol(i, j),
// minres(lambda, lambda, ...) -- compile and run unchanged on the B200.  The
// device state lives in contexts cached by the objects' identities (Q/D pointers, the
// hierarchy, the preconditioner's factor storage), not in the structs, whose layout is the
// reference's.
//
// The generic minres(apply_A, apply_Pinv, ...) (minres.hpp:29-33) still runs its loop on the
// host around device applications.  The overload below runs the whole loop on the device
// (one CUDA graph); it is the call gauss_newton makes after the one-line patch of
// inversion.cpp:261-265 shown in INTEGRATION.md.
#pragma once

#include <span>
#include <utility>

#include "ertinv/inversion.hpp"
#include "ertinv/minres.hpp"

namespace ertinv {

std::pair<Vector, MinresReport> minres(const SaddleOperator& op, const WoodburyPreconditioner& pc,
                                       std::span<const double> b, std::span<const double> x0, double tol,
                                       std::size_t maxit);

// Frees every cached device context (they are otherwise kept for the objects' lifetime).
void gnw_release_contexts();

}  // namespace ertinv
