/* TEST INFRASTRUCTURE ONLY (oracle).  Plain-C descriptors shared by the
 * fp64 oracle (liboracle.so) and the reference-tape gradient oracle
 * (oracle/_ref/libref.so).  They mirror the device descriptors in
 * include/diffmpm.h field for field (in double precision). */
#ifndef ORACLE_CAPI_TYPES_H
#define ORACLE_CAPI_TYPES_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dims[3];
  double dx, dt;
  double gravity[3];
  int boundary; /* 0 slip (mpm.hpp:296-302), 1 sticky */
  double alpha_c, mu_b; /* CouplingParams, mpm.hpp:134-137 */
} OrSim;

typedef struct {
  int kind; /* 0 fixed-corotated, 1 neo-Hookean, 2 elastoplastic, 3 fluid */
  double youngs, poisson, density, volume, yield_stress;
  int wide_yield;
  double viscosity, act_strength, bulk;
} OrMat;

typedef struct {
  int kind; /* 0 plane, 1 sphere, 2 box, 3 cylinder, 4 hollow box */
  double center[3], velocity[3], omega[3], normal[3];
  double radius, half[3], length, thickness;
} OrCol;

typedef struct {
  int kind; /* 0 |com_T - target|^2, 1 -sum mean_z, 2 sum var_z, 3 fluid move */
  double target[3];
  double spill_half, spill_temp;
  double tier_threshold, tier_low, tier_high;
} OrLoss;

#ifdef __cplusplus
}
#endif
#endif
