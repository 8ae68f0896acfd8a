/*
 * One quantum step of a Shor attempt (shor.py:98-117) from plain C through
 * the register handle of libshorb200.so: modexp -> measure -> QFT -> sample.
 * The draws u2, u3 are what the reference's Sampler would return
 * (qstate.py:99 and :113); the host keeps the PCG64 stream.
 *
 *   c_attempt_demo n x w u2 u3 [shards]
 *
 * `shards` > 1 repeats device 0 that many times (the sharded code path on a
 * single GPU).  Prints one JSON line.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "shorb200.h"

#define CHECK(call)                                                          \
    do {                                                                     \
        int rc_ = (call);                                                    \
        if (rc_ != SHB_OK) {                                                 \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, shb_last_error()); \
            return 1;                                                        \
        }                                                                    \
    } while (0)

int main(int argc, char **argv)
{
    if (argc < 6) {
        fprintf(stderr, "usage: %s n x w u2 u3 [shards]\n", argv[0]);
        return 2;
    }
    const uint64_t n = strtoull(argv[1], NULL, 10), x = strtoull(argv[2], NULL, 10);
    const uint32_t w = (uint32_t)strtoul(argv[3], NULL, 10);
    const double u2 = strtod(argv[4], NULL), u3 = strtod(argv[5], NULL);
    const int shards = argc > 6 ? atoi(argv[6]) : 1;
    int devs[16] = {0};
    if (shards < 1 || shards > 16) return 2;

    shb_ctx *reg = NULL;
    CHECK(shb_init_devices(devs, shards, &reg));
    CHECK(shb_ctx_modexp(reg, x, n, w));
    uint32_t k = 0;
    uint64_t M = 0, m = 0;
    double amp = 0.0, norm = 0.0, row[2] = {0.0, 0.0};
    CHECK(shb_measure(reg, u2, &k, &M, &amp));
    CHECK(shb_ctx_dft(reg, SHB_FP64, 1));
    CHECK(shb_norm(reg, &norm));
    CHECK(shb_sample(reg, u3, &m));
    CHECK(shb_copy_spectrum(reg, m, m + 1, row));
    uint64_t bits;
    memcpy(&bits, &amp, sizeof bits);
    printf("{\"k\": %u, \"M\": %llu, \"amp_bits\": \"%016llx\", \"norm\": %.17g, \"m\": %llu, "
           "\"row_m\": [%.17g, %.17g]}\n",
           k, (unsigned long long)M, (unsigned long long)bits, norm, (unsigned long long)m, row[0], row[1]);
    shb_free(reg);
    return 0;
}
