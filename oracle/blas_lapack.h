// TEST INFRASTRUCTURE (oracle only). Prototypes for the CBLAS / LAPACKE entry
// points exported by the OpenBLAS 0.3.15 bundled in this image
// (opencv_python_headless.libs/libopenblasp-r0-59ffcd50.3.15.so, 32-bit ints,
// unprefixed symbols). The image has no cblas.h / lapacke.h, so the oracle
// declares exactly what it uses.
#pragma once

extern "C" {
enum { kCblasColMajor = 102 };
enum { kCblasNoTrans = 111, kCblasTrans = 112 };
enum { kCblasUpper = 121, kCblasLower = 122 };
enum { kCblasNonUnit = 131, kCblasUnit = 132 };
enum { kCblasLeft = 141, kCblasRight = 142 };

void cblas_dgemm(int order, int ta, int tb, int m, int n, int k, double alpha, const double* a,
                 int lda, const double* b, int ldb, double beta, double* c, int ldc);
void cblas_dgemv(int order, int ta, int m, int n, double alpha, const double* a, int lda,
                 const double* x, int incx, double beta, double* y, int incy);
void cblas_dtrsm(int order, int side, int uplo, int ta, int diag, int m, int n, double alpha,
                 const double* a, int lda, double* b, int ldb);

#define kLapackColMajor 102
int LAPACKE_dgeqrf(int layout, int m, int n, double* a, int lda, double* tau);
int LAPACKE_dorgqr(int layout, int m, int n, int k, double* a, int lda, const double* tau);
int LAPACKE_dgesdd(int layout, char jobz, int m, int n, double* a, int lda, double* s, double* u,
                   int ldu, double* vt, int ldvt);
int LAPACKE_dsyevd(int layout, char jobz, char uplo, int n, double* a, int lda, double* w);
int LAPACKE_dpotrf(int layout, char uplo, int n, double* a, int lda);
int LAPACKE_dpotrs(int layout, char uplo, int n, int nrhs, const double* a, int lda, double* b,
                   int ldb);
int LAPACKE_dgeqp3(int layout, int m, int n, double* a, int lda, int* jpvt, double* tau);

void openblas_set_num_threads(int n);
int openblas_get_num_threads(void);
char* openblas_get_corename(void);
}
