/* TEST INFRASTRUCTURE ONLY: hidden-visibility sin/cos/sincos for the
 * reference build (oracle/_ref).  References from the reference objects bind
 * to these at link time, so the reference uses the same portable sin/cos as
 * the oracle and the kernels (pbo_math.h pbm_sincos). */
#define _GNU_SOURCE
#include "pbo_math.h"

double sin(double x) { double s, c; pbm_sincos(x, &s, &c); return s; }
double cos(double x) { double s, c; pbm_sincos(x, &s, &c); return c; }
void sincos(double x, double* s, double* c) { pbm_sincos(x, s, c); }
