// The staged record walk's launch (staged_kernel.cuh); instances in k_st_b*.cu.
#include <cuda_runtime.h>

#include <cstdlib>

#include "escs_internal.h"
#include "staged_kernel.cuh"

namespace escs {
namespace kern {

// per-lane-map instance tables (k_st_b*.cu)
StagedFn get_staged_b32(int h, int npw, bool probe);
StagedFn get_staged_b64(int h, int npw, bool probe);
StagedFn get_staged_b128(int h, int npw, bool probe);
StagedFn get_staged_b128_f8(int h, int npw, bool probe);

StagedFn get_staged(int n, int F, int h, int npw, bool probe) {
    if (n == 32 && F == 4) return get_staged_b32(h, npw, probe);
    if (n == 64 && F == 4) return get_staged_b64(h, npw, probe);
    if (n == 128 && F == 4) return get_staged_b128(h, npw, probe);
    if (n == 128 && F == 8) return get_staged_b128_f8(h, npw, probe);
    return nullptr;
}

}  // namespace kern

bool staged_supported(int h, int bcols, int colf, int npw) {
    return kern::get_staged(bcols, colf, h, npw, false) != nullptr;
}

size_t staged_smem_bytes(const DevPlan& dp) {
    return ((size_t)dp.st_sb_floats + (size_t)dp.st_sr_words + (size_t)dp.st_max_stages * dp.st_hs) * 4;
}

int launch_staged(const DevPlan& dp, const float* rec, const float* B, float* C, void* stream, bool probe) {
    kern::StagedFn fn = kern::get_staged(dp.bcols, dp.colf, dp.h, dp.st_npw, probe);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    if (dp.st_n_cta == 0) return 0;
    const size_t smem = staged_smem_bytes(dp);
    kern::SParams p = {};
    p.cta = reinterpret_cast<const int4*>(dp.st_cta);
    p.stage = reinterpret_cast<const int4*>(dp.st_stage);
    p.hdr = dp.st_hdr;
    p.rec = reinterpret_cast<const int*>(rec);
    p.B = B;
    p.C = dp.st_nsplit > 1 ? dp.st_ws : C;
    p.m = dp.m;
    p.n = dp.bcols;
    p.hs = dp.st_hs;
    p.nslot = dp.st_warps * dp.st_npw;
    p.sb_floats = dp.st_sb_floats;
    p.sr_words = dp.st_sr_words;
    p.split_stride = dp.st_nsplit > 1 ? (long long)dp.m * dp.bcols : 0;
    p.Cout = C;
    p.counters = dp.st_counters;
    p.nsplit = dp.st_nsplit;
    p.coop = (!probe && dp.st_nsplit > 1 && dp.st_coop) ? 1 : 0;
    if (probe) p.C = C;   // the sink
    p.rows_per_block = dp.st_warps * dp.st_npw * dp.h;
    p.max_st = dp.st_max_stages;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(dp.st_n_cta);
    cfg.blockDim = dim3(32 * dp.st_warps);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (dp.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    static const bool coop_attr = [] {
        const char* e = std::getenv("ESCS_ST_COOPATTR");
        return !(e && e[0] == '0');
    }();
    if (p.coop && coop_attr) {   // the split combine spins on its row block's CTAs: all must be resident
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, fn, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return (int)e;
    }
    if (!probe && dp.st_nsplit > 1 && !p.coop) {
        const long long n4 = (long long)dp.m * dp.bcols / 4;
        cudaLaunchConfig_t rc = cfg;
        rc.blockDim = dim3(128);
        rc.dynamicSmemBytes = 0;
        rc.numAttrs = dp.pdl ? 1 : 0;
        long long blocks = (n4 + 127) / 128;
        if (blocks > 148LL * 16) blocks = 148LL * 16;
        rc.gridDim = dim3((unsigned)blocks);
        e = cudaLaunchKernelEx(&rc, kern::esc_staged_reduce_kernel<0>, (const float*)dp.st_ws, C, n4, n4,
                               dp.st_nsplit);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return (int)e;
        }
    }
    return (int)cudaGetLastError();
}

// Kernel attributes are per function and shared by every plan: set the
// dynamic shared-memory limit once, to the most the function can take (the
// device's opt-in per-block maximum less its static shared memory), so no
// plan ever lowers it under another.
int staged_blocks_per_sm(const DevPlan& dp) {
    kern::StagedFn fn = kern::get_staged(dp.bcols, dp.colf, dp.h, dp.st_npw, false);
    int nb = 0;
    if (!fn || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)fn, 32 * dp.st_warps,
                                                             staged_smem_bytes(dp)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nb;
}

int prepare_staged(const DevPlan& dp) {
  for (int probe = 0; probe < 2; probe++) {
    kern::StagedFn fn = kern::get_staged(dp.bcols, dp.colf, dp.h, dp.st_npw, probe == 1);
    if (!fn) return (int)cudaErrorInvalidConfiguration;
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes attr;
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&attr, (const void*)fn);
    if (e != cudaSuccess) return (int)e;
    const int cap = optin - (int)attr.sharedSizeBytes;
    {   // the shared-memory carveout at its maximum (the walk's B rows and records
        // live there, L1 holds nothing it reuses): no reconfiguration between launches
        static const int carve = [] {
            const char* c = std::getenv("ESCS_ST_CARVEOUT");
            return c ? std::atoi(c) : 100;
        }();
        if (carve >= 0) {
            e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            if (e != cudaSuccess) return (int)e;
        }
    }
    if ((int)staged_smem_bytes(dp) > cap) return (int)cudaErrorInvalidConfiguration;
    if (attr.maxDynamicSharedSizeBytes >= cap) continue;
    e = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    if (e != cudaSuccess) return (int)e;
  }
  return 0;
}

}  // namespace escs
