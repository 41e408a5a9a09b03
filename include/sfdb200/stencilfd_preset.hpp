// The B200 backend under the reference's own operator API, unchanged.
//
// A caller of stencilfd (/root/reference/proj) keeps calling
//     sfd::seismic::forward / adjoint / gradient, sfd::verify::adjoint_test, ...
// and selects the GPU through RunConfig::preset, the knob those calls already
// take (seismic.hpp:85-89, seismic.cpp:65-70):
//
//     sfd::seismic::RunConfig cfg;
//     cfg.preset = sfdb200::stencilfd_preset("/path/to/this/repo");
//     auto fwd = sfd::seismic::forward(model, src, trace, rec, nt, dt, true, cfg);
//
// runtime::compile_and_load then compiles every generated kernel through
// bin/sfdb200-jit (gcc's -wrapper), which swaps the loop nest for a shim
// forwarding `<Name>_call(argv)` to sfdb200_call with the descriptor read
// back from the source (csrc/jit.cpp); the shim links libsfdb200.so
// (`-Wl,--no-as-needed`: the reference's command puts the preset flags before
// the source file, runtime.cpp:213-214, so a plain `-lsfdb200` would be
// dropped by --as-needed).  Nothing in the reference changes.
//
// desc_of() is the same descriptor computed from the KernelIR directly, for a
// caller that bypasses the JIT.
#pragma once

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../sfdb200.h"
#include "stencilfd/lowering.hpp"
#include "stencilfd/runtime.hpp"

namespace sfdb200 {

/// root: the directory holding include/ and paper_1608_08658_b200/ (default
/// $SFDB200_ROOT); device: the CUDA ordinal the shims bind.
inline sfd::runtime::CompilerPreset stencilfd_preset(std::string root = "", int device = 0) {
    if (root.empty()) {
        const char* env = std::getenv("SFDB200_ROOT");
        if (!env || !*env) throw std::invalid_argument("sfdb200: set SFDB200_ROOT or pass the root");
        root = env;
    }
    const std::string pkg = root + "/paper_1608_08658_b200";
    return {"b200",
            {"-O2", "-wrapper", pkg + "/bin/sfdb200-jit", "-DSFDB200_DEVICE=" + std::to_string(device),
             "-L" + pkg, "-Wl,--no-as-needed", "-lsfdb200", "-Wl,-rpath," + pkg}};
}

/// The descriptor of a kernel built by seismic::build_{forward,adjoint,
/// gradient}_ir (seismic.cpp:241-331): what the generated source bakes in.
/// dt and h are the values given to the builder (they only appear folded
/// into the IR's constants); save: the forward history flag.
inline sfdb200_desc desc_of(const sfd::lower::KernelIR& ir, double dt, double h, bool save = false,
                            int device = 0) {
    sfdb200_desc d{};
    if (ir.find_grid("grad")) {
        d.kind = SFDB200_GRADIENT;
        d.flags = SFDB200_F_GRAD_NO_ROW2;  // seismic::gradient adds t = 2 on the host
    } else if (ir.find_grid("v")) {
        d.kind = SFDB200_ADJOINT;
    } else if (ir.find_grid("u")) {
        d.kind = SFDB200_FORWARD;
        d.save = save ? 1 : 0;
    } else {
        throw std::invalid_argument("sfdb200: not a seismic operator kernel");
    }
    d.ndim = ir.ndim();
    for (int k = 0; k < d.ndim; ++k) d.padded[k] = ir.extents[static_cast<std::size_t>(k)];
    d.space_order = static_cast<int>(2 * ir.halo);
    d.nt = ir.nt;
    d.dt = dt;
    d.h = h;
    for (const sfd::lower::SparseSet& s : ir.sparse_sets) (s.name == "src" ? d.nsrc : d.nrec) = s.npoints;
    d.device = device;
    return d;
}

}  // namespace sfdb200
