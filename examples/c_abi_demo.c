/* Plain-C use of libshorb200 through include/shorb200.h only (no Python, no
 * torch): the QFT of a collapsed Shor register via the host-buffer drop-in of
 * qft.dense_dft, and the _kernels.partial_row_sums seam.
 *
 *   gcc -O2 -I include examples/c_abi_demo.c -L paper_1801_01434_b200 \
 *       -Wl,-rpath,$PWD/paper_1801_01434_b200 -lshorb200 -lm -o c_abi_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "shorb200.h"

int main(void)
{
    /* n = 15, x = 2, q = 256, outcome k = 1: support {0, 4, ..., 252}, amplitude 1/8
     * (SPEC.md:163); the exact peak law says |V|^2 = 1/4 at {0, 64, 128, 192}. */
    const uint64_t q = 256;
    double *state = calloc(2 * q, sizeof(double)), *out = calloc(2 * q, sizeof(double));
    for (uint64_t a = 0; a < q; a += 4) state[2 * a] = 0.125;
    int rc = shb_dense_dft_host(state, q, 1, SHB_FP64, out);
    if (rc != SHB_OK) {
        fprintf(stderr, "shb_dense_dft_host: %s\n", shb_last_error());
        return 1;
    }
    double worst = 0.0, off = 0.0;
    for (uint64_t c = 0; c < q; c++) {
        const double p = out[2 * c] * out[2 * c] + out[2 * c + 1] * out[2 * c + 1];
        if (c % 64 == 0) worst = fmax(worst, fabs(p - 0.25));
        else off = fmax(off, p);
    }
    /* the seam: rows 64..67 over inputs [0, q), unscaled -> row 64 = 64 * 0.125 = 8 */
    double rows[8];
    rc = shb_partial_row_sums_host(rows, state, NULL, q, 64, 68, 0, q);
    if (rc != SHB_OK) {
        fprintf(stderr, "shb_partial_row_sums_host: %s\n", shb_last_error());
        return 1;
    }
    /* argument errors come back as status codes, never as aborts */
    const int bad = shb_dense_dft_host(state, 100, 1, SHB_FP64, out);
    printf("peaks |p-1/4| <= %.3g, off-peak p <= %.3g, row64 = %.15g, bad q -> %d (%s)\n", worst, off, rows[0],
           bad, shb_last_error());
    const int ok = worst < 1e-12 && off < 1e-24 && fabs(rows[0] - 8.0) < 1e-12 && bad == SHB_EINVAL;
    free(state);
    free(out);
    return ok ? 0 : 2;
}
