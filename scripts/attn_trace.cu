// Timeline of one flash-attention CTA (CTA 0 = the longest query-tile pair): build with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DBZ_ATTN_TRACE -I include \
//        -o attn_trace scripts/attn_trace.cu paper_2412_17246_b200/csrc/runtime.cpp ... (see call script)
#include "../paper_2412_17246_b200/csrc/attention_tcgen05.cu"
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int B = 4, S = 2000, H = 32, KV = 32, hd = 128;
  const int ld = (H + 2 * KV) * hd;
  std::vector<uint16_t> h(static_cast<size_t>(B) * S * ld);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    float f = ((x >> 8) / 16777216.0f - 0.5f) * 2.0f;
    uint32_t bits;
    memcpy(&bits, &f, 4);
    v = static_cast<uint16_t>(bits >> 16);
  }
  void *qkv, *out, *ws;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&out, static_cast<size_t>(B) * S * H * hd * 2);
  int64_t need = 0;
  bz_prefill_attention_workspace_bytes(B, S, KV, hd, &need);
  cudaMalloc(&ws, need);
  for (int it = 0; it < 3; ++it) {
    int rc = bz_prefill_attention(qkv, ld, B, S, H, KV, hd, ws, need, out, H * hd, nullptr);
    if (rc) { printf("rc=%d %s\n", rc, bz_last_error()); return 1; }
  }
  cudaDeviceSynchronize();
  std::vector<unsigned long long> tr(4096);
  cudaMemcpyFromSymbol(tr.data(), bz::attn::g_trace, 4096 * 8);
  unsigned long long t0 = ~0ull;
  for (auto v : tr) if (v && v < t0) t0 = v;
  const int nj = 16;  // CTA 0 = pair 7 of S=2000: key tiles 0..15
  printf("j  | A: wait_s  got_s  p_full | B: wait_s  got_s  p_full | MMA: A wait_p got_p  B wait_p got_p (ns from first stamp)\n");
  for (int j = 0; j < nj; ++j) {
    auto f = [&](int i) { return tr[i] ? static_cast<long long>(tr[i] - t0) : -1ll; };
    printf("%2d | %7lld %7lld %7lld | %7lld %7lld %7lld | %7lld %7lld %7lld %7lld\n", j, f(4 * j), f(4 * j + 1),
           f(4 * j + 2), f(1024 + 4 * j), f(1024 + 4 * j + 1), f(1024 + 4 * j + 2), f(2048 + 8 * j), f(2048 + 8 * j + 1),
           f(2048 + 8 * j + 2), f(2048 + 8 * j + 3));
  }
  return 0;
}
