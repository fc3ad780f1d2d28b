/* c_client.c -- a plain C caller of the AutoSAGE-B200 C-ABI (include/autosage_b200.h).
 *
 * The reference's worked SpMM example (proj/tests/test_kernels.cpp:50-70):
 * A = [[0, 2], [0, 0]], B = [[1, 1], [3, 4]]  ->  C = [[6, 8], [0, 0]],
 * through the baseline, a fixed variant, the scheduler (spmm_auto with a
 * schedule cache) and the async host pipeline.  Exit 0 iff every result matches.
 *
 *   gcc -std=c11 -I include examples/c_client.c -L paper_2511_17594_b200 \
 *       -lautosage_b200 -Wl,-rpath,$PWD/paper_2511_17594_b200 -o c_client
 */
#include <stdio.h>
#include <string.h>

#include "autosage_b200.h"

static int check(const char* what, const float* c) {
    const float want[4] = {6.f, 8.f, 0.f, 0.f};
    if (memcmp(c, want, sizeof want) != 0) {
        fprintf(stderr, "%s: got [[%g, %g], [%g, %g]]\n", what, c[0], c[1], c[2], c[3]);
        return 1;
    }
    return 0;
}

#define TRY(call)                                                       \
    do {                                                                \
        if ((call) != AS_OK) {                                          \
            fprintf(stderr, "%s failed: %s\n", #call, as_last_error()); \
            return 1;                                                   \
        }                                                               \
    } while (0)

int main(void) {
    const uint64_t rowptr[3] = {0, 1, 1};
    const uint32_t colind[1] = {1};
    const float val[1] = {2.f};
    const float b[4] = {1.f, 1.f, 3.f, 4.f};
    float c[4];
    int bad = 0;

    as_graph g;
    TRY(as_graph_create(rowptr, colind, val, 2, 2, 1, 0, &g));

    as_kernel_result r;
    TRY(as_spmm_host(NULL, g, b, 2, 2, c, &r)); /* NULL variant: baseline kernel */
    bad |= check("baseline", c);

    as_variant v;
    TRY(as_variant_from_string("spmm:hubsplit:ft=32:rpc=4:vec=1:hubt=1", &v));
    memset(c, 0, sizeof c);
    TRY(as_spmm_host(&v, g, b, 2, 2, c, &r));
    bad |= check("hubsplit", c);

    memset(c, 0, sizeof c);
    TRY(as_spmm_host_async(&v, g, b, 2, 2, c, &r));
    TRY(as_graph_synchronize(g));
    bad |= check("async", c);

    /* scheduler on device buffers: the library's host forms stage through the
     * graph; here decide + run through the host entry with the chosen variant */
    as_cache cache;
    TRY(as_cache_create(&cache));
    as_context ctx;
    memset(&ctx, 0, sizeof ctx);
    ctx.cache = cache;
    as_probe_config cfg;
    as_probe_config_default(&cfg);
    cfg.iters = 2;
    float *b_dev = NULL, *c_dev = NULL;
    TRY(as_host_alloc((void**)&b_dev, sizeof b)); /* pinned host memory is device-addressable */
    TRY(as_host_alloc((void**)&c_dev, sizeof c));
    memcpy(b_dev, b, sizeof b);
    as_decision d;
    TRY(as_spmm_auto(&ctx, &cfg, g, b_dev, 2, 2, c_dev, &d));
    TRY(as_graph_synchronize(g));
    bad |= check("spmm_auto", c_dev);
    uint64_t n = 0;
    TRY(as_cache_size(cache, &n));
    if (n != 1) {
        fprintf(stderr, "cache holds %llu records\n", (unsigned long long)n);
        bad = 1;
    }
    char name[128] = "baseline";
    if (d.has_choice) TRY(as_variant_to_string(&d.choice, name, sizeof name));
    printf("spmm_auto chose %s (%llu kernel launches so far)\n", name,
           (unsigned long long)as_kernel_launch_count());

    as_host_free(b_dev);
    as_host_free(c_dev);
    as_cache_destroy(cache);
    as_graph_destroy(g);
    printf(bad ? "FAIL\n" : "OK\n");
    return bad;
}
