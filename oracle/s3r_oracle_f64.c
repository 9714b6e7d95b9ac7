/*
 * s3r_oracle_f64.c — fp64 SHADOW instance of the CPU oracle (libm exp).
 * TEST INFRASTRUCTURE ONLY (see s3r_oracle.h).  Same algorithm text as the
 * fp32 contract (s3r_oracle_impl.inc), evaluated in double precision; the pin
 * tests use it to bound the fp32 contract's rounding error.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "s3r_oracle.h"

double so_exp_f64(double x) { return exp(x); }

#define REAL double
#define SO(x) x##_f64
#define R(x) x
#define FMA fma
#define SQRT sqrt
#define CEIL ceil
#define FLOOR floor
#define FMIN fmin
#define FMAX fmax
#define ISFIN isfinite
#define EXPF exp
#include "s3r_oracle_impl.inc"
