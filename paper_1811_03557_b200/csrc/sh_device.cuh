// Device-side real spherical harmonics (R8: orthonormal, no Condon-Shortley phase, ν = l^2 + l + m),
// by the fully-normalised associated-Legendre recurrence in Cartesian form (pole-safe):
//   P̂_m^m = P̂_{m-1}^{m-1} sqrt((2m+1)/(2m)),  P̂_{m+1}^m = z sqrt(2m+3) P̂_m^m,
//   P̂_l^m = a_lm (z P̂_{l-1}^m - b_lm P̂_{l-2}^m),  a = sqrt((4l^2-1)/(l^2-m^2)),
//   b = sqrt(((l-1)^2-m^2)/(4(l-1)^2-1));  C_m + i S_m = (x + i y)^m.
//   Y_l0 = P̂_l^0,  Y_lm = sqrt2 P̂_l^m C_m,  Y_l,-m = sqrt2 P̂_l^m S_m.
// emit(nu, value) is called once per (l, m).
#pragma once

template <typename Emit>
__device__ __forceinline__ void real_sh_unit(double x, double y, double z, int lmax, Emit&& emit) {
  double pmm = 0.28209479177387814347;   // 1/sqrt(4 pi)
  double Cm = 1.0, Sm = 0.0;
  for (int m = 0; m <= lmax; ++m) {
    if (m > 0) {
      pmm *= sqrt((2.0 * m + 1.0) / (2.0 * m));
      const double Cn = x * Cm - y * Sm, Sn = x * Sm + y * Cm;
      Cm = Cn;
      Sm = Sn;
    }
    double p2 = 0.0, p1 = pmm;
    for (int l = m; l <= lmax; ++l) {
      double pl;
      if (l == m) pl = pmm;
      else if (l == m + 1) pl = z * sqrt(2.0 * m + 3.0) * pmm;
      else {
        const double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
        const double b = sqrt(((l - 1.0) * (l - 1.0) - (double)m * m) / (4.0 * (l - 1.0) * (l - 1.0) - 1.0));
        pl = a * (z * p1 - b * p2);
      }
      if (l > m) { p2 = p1; p1 = pl; }
      if (m == 0) {
        emit(l * l + l, pl);
      } else {
        emit(l * l + l + m, 1.41421356237309504880 * pl * Cm);
        emit(l * l + l - m, 1.41421356237309504880 * pl * Sm);
      }
    }
  }
}
