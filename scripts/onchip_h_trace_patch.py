import sys
p='/root/repo/paper_2503_08467_b200/csrc/expert_mlp.cu'
s=open(p).read()
def rep(a,b):
    global s
    assert a in s, a[:80]
    s=s.replace(a,b,1)
rep('''struct MlpArgs {''','''__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ unsigned long long g_trace[64 * 64];
struct MlpArgs {''')
rep('''  const uint32_t j = cluster_ctarank();''','''  const uint32_t j = cluster_ctarank();
  unsigned long long* tr = blockIdx.x < 64 ? g_trace + blockIdx.x * 64 : nullptr;
  if (tr && threadIdx.x == 0) { for (int q = 0; q < 64; ++q) tr[q] = 0; tr[0] = gt(); }''')
rep('''  griddep_launch_dependents();
  const uint32_t tmem = *tmem_slot;''','''  griddep_launch_dependents();
  if (tr && threadIdx.x == 0) tr[1] = gt();
  const uint32_t tmem = *tmem_slot;''')
rep('''        for (int kb = 0; kb < nkb_up; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();''','''        for (int kb = 0; kb < nkb_up; ++kb) {
          mbar_wait(&full[s], ph);
          if (tr && lane == 0 && kb == 0 && i < 3) tr[2 + i * 8] = gt();
          tc_fence_after();''')
rep('''        if (elect_one()) mma_commit(&upfull[b]);''','''        if (tr && lane == 0 && i < 3) tr[3 + i * 8] = gt();
        if (elect_one()) mma_commit(&upfull[b]);''')
rep('''        mbar_wait(hfull, par);            // every slice of this unit's H is in this CTA''','''        mbar_wait(hfull, par);            // every slice of this unit's H is in this CTA
        if (tr && lane == 0 && i - 1 < 3) tr[4 + (i - 1) * 8] = gt();''')
rep('''        if (elect_one()) {
          mma_commit(dnfull);''','''        if (tr && lane == 0 && i - 1 < 3) tr[5 + (i - 1) * 8] = gt();
        if (elect_one()) {
          mma_commit(dnfull);''')
rep('''      mbar_wait(hempty, (k & 1) ^ 1);   // every CTA's down MMAs of the previous unit are done
      tc_fence_after();''','''      mbar_wait(hempty, (k & 1) ^ 1);   // every CTA's down MMAs of the previous unit are done
      if (tr && threadIdx.x == 128 && k < 3) tr[6 + k * 8] = gt();
      tc_fence_after();''')
rep('''        mbar_arrive(&uptempty[b]);
        mbar_arrive(hfull);
      }''','''        mbar_arrive(&uptempty[b]);
        mbar_arrive(hfull);
      }
      if (tr && threadIdx.x == 128 && k < 3) tr[7 + k * 8] = gt();''')
rep('''      mbar_wait(dnfull, k & 1);
      tc_fence_after();''','''      mbar_wait(dnfull, k & 1);
      if (tr && threadIdx.x == 256 && k < 3) tr[8 + k * 8] = gt();
      tc_fence_after();''')
rep('''      if (lane == 0) mbar_arrive(dntempty);
    }''','''      if (lane == 0) mbar_arrive(dntempty);
      if (tr && threadIdx.x == 256 && k < 3) tr[9 + k * 8] = gt();
    }
    if (tr && threadIdx.x == 256) tr[40] = gt();''')
rep('''bool expert_mlp_supported(int h, int F, int E) {''','''void mlp_trace_dump() {
  static unsigned long long h[64 * 64];
  cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
  for (int b = 0; b < 64; b += 4) {
    unsigned long long t0 = h[b * 64];
    printf("cta %2d: griddep %4llu |", b, (h[b * 64 + 1] - t0) / 100);
    for (int u = 0; u < 3; ++u) {
      printf(" u%d:", u);
      for (int q = 2; q < 10; ++q) {
        unsigned long long v = h[b * 64 + q + u * 8];
        printf(" %4lld", v ? (long long)(v - t0) / 100 : -1LL);
      }
    }
    printf(" | end %lld\\n", (long long)(h[b * 64 + 40] - t0) / 100);
  }
}

bool expert_mlp_supported(int h, int F, int E) {''')
s=s.replace('#include <algorithm>\n','#include <algorithm>\n#include <cstdio>\n',1)
open(p,'w').write(s)
p='/root/repo/paper_2503_08467_b200/csrc/moeshard.cu'
s=open(p).read()
s=s.replace('''int moeshard_destroy(moeshard_ctx* c) {''','''int moeshard_mlp_trace(void) { cudaDeviceSynchronize(); moeshard::mlp_trace_dump(); return 0; }

int moeshard_destroy(moeshard_ctx* c) {''')
s=s.replace('''using namespace moeshard;
''','''namespace moeshard { void mlp_trace_dump(); }
using namespace moeshard;
''',1)
open(p,'w').write(s)
