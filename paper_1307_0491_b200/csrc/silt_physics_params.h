// silt_physics_params.h — per-launch physical parameters (host + device).
#pragma once

namespace silt_dev {

// error bits raised on device (mapped to the reference's exceptions on host)
constexpr unsigned kErrNegDepth = 1u;  // check_depth (src/stepper.cpp:91-100)
constexpr unsigned kErrRiemann = 2u;   // interface_riemann (src/riemann.cpp:332-337)
constexpr unsigned kErrDry = 4u;       // cfl_dt all dry (src/stepper.cpp:56)
constexpr unsigned kErrPeer = 8u;      // multi-process strips: a peer rank missed a step
                                       // (no reference analogue: run_parallel's workers
                                       // share one process; a dead worker rethrows)

// Physics (include/silt/physics.hpp:7-11) + bedload law (bedload.hpp:32-52) +
// the interface safety factor (Scenario::safety, scenarios.hpp:47).
struct Params {
    double g, h_dry, a_g, m_g, safety, half_g;
    int m3;        // m_g == 3: closed-form Grass terms in the FAST variant
    int shields;   // BedloadLaw::Kind::Shields (kernels are instantiated per kind)
    int formula;   // ShieldsFormula, enum order of bedload.hpp:12-18
    int friction;  // FrictionModel: 0 Darcy-Weisbach, 1 Manning
    double tau_cr, d_s, rel_density, fcoef;
    double scale;  // sqrt((s - 1) * g * d * d * d)        (src/bedload.cpp:161)
    double ktau;   // FAST: tau = ktau s^2 [h^(-1/3) for Manning]
};

}  // namespace silt_dev
