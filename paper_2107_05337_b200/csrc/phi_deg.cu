// One spline degree of the Phi kernels: compiled once per degree with
// -DPHI_DEG=<1..8> (see build.py), so the eight instantiations build in
// parallel.  The device code is in phi_device.cuh.
#include "phi_device.cuh"

#ifndef PHI_DEG
#error "compile with -DPHI_DEG=<degree>"
#endif

namespace phi {
template struct DegLaunch<PHI_DEG>;
}  // namespace phi
