// hydro_internal.h -- private declarations shared by the library's translation units.
#ifndef HYDRO_INTERNAL_H_
#define HYDRO_INTERNAL_H_

#include <stdint.h>

#define HYDRO_MAXN 4  // H1 nodes per dim (k <= 3)
#define HYDRO_MAXQ 6  // Gauss-Legendre points per dim
#define HYDRO_TAB_DOUBLES 128  // packed device tables: w[q] B[q][n] G[q][n] Bl[q][m] <= 6+24+24+18

typedef struct {
  int k, q;
  double xi[HYDRO_MAXQ], w[HYDRO_MAXQ];
  double B[HYDRO_MAXQ][HYDRO_MAXN];      // l_a(xi_q), GLL Lagrange, degree k
  double G[HYDRO_MAXQ][HYDRO_MAXN];      // l_a'(xi_q)
  double Bl[HYDRO_MAXQ][HYDRO_MAXN - 1]; // GL Lagrange, degree k-1
} hydro_tables_t;

// tables.cpp (host, binary128): returns 0 on success.
int hydro_make_tables(int k, int q, hydro_tables_t *T);

// Device status block (one per context / per sample plan instance).
typedef struct {
  unsigned long long dt_key;     // order-preserving key of the running dt minimum
  unsigned long long first_bad;  // lowest tangled element (sticky), ~0ull if none
  unsigned int nan_flag;         // this call: some dt_q was NaN
  unsigned int nan_sticky;       // sticky until status_sync
} hydro_devstatus;

#endif  // HYDRO_INTERNAL_H_
