/* bm_oracle.h — CPU restatement of the reference path. TEST INFRASTRUCTURE ONLY
 * (see bm_oracle.c header).  Records use the ABI's bm_patch_record layout so
 * oracle and GPU outputs compare field by field. */
#ifndef BM_ORACLE_H
#define BM_ORACLE_H
#include <stdint.h>
#include "../include/blockmend_b200.h"

typedef bm_patch_record orc_record;
#define ORC_FALLBACK BM_REC_FALLBACK
#define ORC_DEFERRED BM_REC_DEFERRED
#define ORC_HAS_NU BM_REC_HAS_NU
#define ORC_HAS_PHI BM_REC_HAS_PHI
#define ORC_HAS_BW BM_REC_HAS_BW
#define ORC_HAS_M BM_REC_HAS_M

typedef struct {
  int layer, fallback, m, has_nu;
  double beta, alpha, nu, gap;
} orc_estimate_info;

/* conceal_image (profiles.py:263-323) on one float64 frame. Returns 0, or 2
 * when LOST pixels remain outside the block grid (profiles.py:305). */
int orc_conceal(int H, int W, const double* pixels, const uint8_t* states, double t_phi, double t_nu,
                double sigma2, int forced_layer, double* out_pixels, orc_record* out_records,
                long max_records, long* out_nrec, long* out_lost_cells);
/* the same with the cells of each dependency level on `threads` threads */
int orc_conceal_dag(int H, int W, const double* pixels, const uint8_t* states, double t_phi, double t_nu,
                    double sigma2, int forced_layer, double* out_pixels, orc_record* out_records,
                    long max_records, long* out_nrec, long* out_lost_cells, int threads);
void orc_brl(const double* y0, int n, double* out4);
/* NumPy's pairwise summation of a[0..n) (test hook for tests/test_oracle_numerics.py) */
double orc_pairwise_sum(const double* a, long n);
int orc_idl(const double* y0, int n, const double* x, const double* y, int m, double sigma2,
            double* out4, double* raw_sum);
int orc_hql(const double* y0, int n, const double* x, const double* y, int m, double sigma2,
            double* out4, orc_estimate_info* info);
#endif
