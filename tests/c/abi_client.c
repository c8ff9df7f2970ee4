/* Plain-C client of libescs.so (include/escs.h): no Python, no torch.
 *   abi_client host   -- host-only plan + export + error codes (no GPU)
 *   abi_client device -- plan, escs_spmm and escs_spmm_group on cudaMalloc'd
 *                        buffers, check C
 * The matrix is the 4x4 worked example of SPEC.md S:123 (golden plan in
 * tests/golden/spec_4x4_plan.json); C = A x B is checked exactly against a
 * hand-computed product.  Exit code 0 = pass. */
#include <stdio.h>
#include <string.h>
#include <cuda_runtime.h>
#include "escs.h"

static const int32_t rowptr[5] = {0, 3, 6, 6, 7};
static const int32_t colidx[7] = {0, 1, 3, 0, 1, 3, 2};

static int check_host(void) {
    escs_params p;
    memset(&p, 0, sizeof p);
    p.ufi = 4; p.T = 4; p.host_only = 1;
    escs_plan_t pl = escs_plan_ex(4, 4, 7, rowptr, colidx, 32, &p);
    if (!pl) { const char* m; escs_last_error(&m); fprintf(stderr, "plan: %s\n", m); return 1; }
    escs_plan_view v;
    if (escs_plan_export(pl, &v) != ESCS_OK) return 2;
    static const int32_t slot[7] = {0, 3, 1, 4, 2, 5, 6}, gcol[4] = {0, 1, 3, 2};
    if (v.header[8] != 2 || v.header[9] != 4 || memcmp(v.slot_src, slot, sizeof slot) ||
        memcmp(v.gcol, gcol, sizeof gcol) || v.grp_mask[0] != 3 || v.grp_mask[1] != 8) return 3;
    if (escs_spmm(pl, NULL, NULL, NULL, NULL) != ESCS_ERR_ARG) return 4;
    escs_free(pl);
    escs_free(NULL);
    static const int32_t bad[7] = {0, 1, 3, 0, 1, 9, 2};          /* column 9 >= k */
    if (escs_plan_ex(4, 4, 7, rowptr, bad, 32, &p) != NULL) return 5;
    const char* msg = NULL;
    if (escs_last_error(&msg) != ESCS_ERR_CSR || !strstr(msg, "row 1")) return 6;
    printf("host ok: %s\n", escs_version());
    return 0;
}

static int check_device(void) {
    const int n = 32;
    float vals[7] = {1, 2, 3, 4, 5, 6, 7}, B[4 * 32], C[4 * 32], ref[4 * 32];
    for (int i = 0; i < 4 * n; i++) B[i] = (float)((i * 7) % 13 - 6);
    memset(ref, 0, sizeof ref);
    for (int i = 0; i < 4; i++)
        for (int t = rowptr[i]; t < rowptr[i + 1]; t++)
            for (int j = 0; j < n; j++) ref[i * n + j] += vals[t] * B[colidx[t] * n + j];
    escs_plan_t pl = escs_plan(4, 4, 7, rowptr, colidx, n);
    if (!pl) { const char* m; escs_last_error(&m); fprintf(stderr, "plan: %s\n", m); return 10; }
    float *dv, *dB, *dC;
    if (cudaMalloc((void**)&dv, sizeof vals) || cudaMalloc((void**)&dB, sizeof B) ||
        cudaMalloc((void**)&dC, sizeof C)) return 11;
    cudaMemcpy(dv, vals, sizeof vals, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xff, sizeof C);                               /* NaN: proves overwrite */
    if (escs_spmm(pl, dv, dB, dC, NULL) != ESCS_OK) return 12;
    if (cudaMemcpy(C, dC, sizeof C, cudaMemcpyDeviceToHost) != cudaSuccess) return 13;
    if (memcmp(C, ref, sizeof C)) return 14;                       /* small integers: exact */
    /* escs_spmm_group: the same problem twice (two plans, two outputs), one call */
    escs_plan_t pl2 = escs_plan(4, 4, 7, rowptr, colidx, n);
    float* dC2;
    if (!pl2 || cudaMalloc((void**)&dC2, sizeof C)) return 15;
    cudaMemset(dC, 0xff, sizeof C);
    cudaMemset(dC2, 0xff, sizeof C);
    escs_plan_t plans[2] = {pl, pl2};
    const float* vs[2] = {dv, dv};
    const float* Bs[2] = {dB, dB};
    float* Cs[2] = {dC, dC2};
    if (escs_spmm_group(2, plans, vs, Bs, Cs, NULL) != ESCS_OK) return 16;
    escs_plan_t same[2] = {pl, pl};
    if (escs_spmm_group(2, same, vs, Bs, Cs, NULL) != ESCS_ERR_ARG) return 17;  /* plan twice */
    for (int o = 0; o < 2; o++) {
        if (cudaMemcpy(C, Cs[o], sizeof C, cudaMemcpyDeviceToHost) != cudaSuccess) return 18;
        if (memcmp(C, ref, sizeof C)) return 19;
    }
    escs_free(pl2);
    cudaFree(dC2);
    escs_free(pl);
    cudaFree(dv); cudaFree(dB); cudaFree(dC);
    printf("device ok\n");
    return 0;
}

int main(int argc, char** argv) {
    int rc = check_host();
    if (rc) return rc;
    if (argc > 1 && !strcmp(argv[1], "device")) return check_device();
    return 0;
}
