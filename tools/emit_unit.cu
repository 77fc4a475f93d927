// Standalone check of the ordered emission's prefix arithmetic: synthetic tile_info /
// block_sums (no hit flags, so nothing is expanded), counters[0] must equal the total;
// with the dense-tile queue on, the queue must also come back empty and reset.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1810_01051_b200/csrc \
//        tools/emit_unit.cu -o /tmp/emit_unit && /tmp/emit_unit
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ unsigned long long g_dbg[1 << 16];
#define RK_EMIT_DEBUG g_dbg
#include "rk_emit.cu"

int main() {
  using namespace rkb;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int bad = 0;
  for (int queue = 0; queue < 2; ++queue)
  for (uint64_t tiles : {1ull, 31ull, 32ull, 100ull, 512ull, 513ull, 4096ull, 32768ull, 131072ull,
                         2097152ull}) {
    std::vector<uint32_t> info(tiles);
    std::vector<unsigned long long> bs((tiles + 255) / 256, 0);
    unsigned long long tot = 0;
    srand(1);
    for (uint64_t i = 0; i < tiles; ++i) {
      // with the queue: about half the tiles "dense" (>= kDeferMin matches, no chunk
      // flagged, so nothing is written: the queue's hand-off and reset are what's tested)
      info[i] = queue && (rand() & 1) ? kDeferMin + rand() % 3000 : rand() % 700;
      bs[i / 256] += info[i];
      tot += info[i];
    }
    uint32_t *d_info, *d_masks;
    unsigned long long *d_bs, *d_cnt;
    cudaMalloc(&d_info, tiles * 4);
    cudaMalloc(&d_masks, 4);
    cudaMalloc(&d_bs, bs.size() * 8);
    cudaMalloc(&d_cnt, 32);
    unsigned long long *d_work, *d_dq;
    cudaMalloc(&d_work, 32);
    cudaMalloc(&d_dq, tiles * 8);
    cudaMemset(d_work, 0, 32);
    cudaMemset(d_dq, 0, tiles * 8);
    int64_t* d_out;
    cudaMalloc(&d_out, 64);
    cudaMemcpy(d_info, info.data(), tiles * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_bs, bs.data(), bs.size() * 8, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(d_cnt, 0, 32);
      if (queue) {
        const unsigned long long one = 1;
        cudaMemcpy(d_cnt + 3, &one, 8, cudaMemcpyHostToDevice);  // the scan's dense flag
      }
      EmitArgs e = {};
      e.tile_info = d_info;
      e.masks = d_masks;
      e.block_sums = d_bs;
      e.num_tiles = tiles;
      e.counters = d_cnt;
      if (queue) {
        e.out = d_out;
        e.cap = 8;
        e.work = d_work;
        e.queue = d_dq;
      }
      cudaError_t err = launch_emit(e, sms, 0);
      if (err == cudaSuccess) err = cudaDeviceSynchronize();
      unsigned long long got[4];
      cudaMemcpy(got, d_cnt, 32, cudaMemcpyDeviceToHost);
      unsigned long long w[4];
      cudaMemcpy(w, d_work, 32, cudaMemcpyDeviceToHost);
      std::vector<unsigned long long> dq(tiles);
      cudaMemcpy(dq.data(), d_dq, tiles * 8, cudaMemcpyDeviceToHost);
      bool clean = w[0] == 0 && w[1] == 0 && w[2] == 0 && w[3] == 0;
      for (auto x : dq) clean = clean && x == 0;
      if (!clean) {
        ++bad;
        printf("queue=%d tiles=%llu rep=%d: queue not reset (%llu %llu %llu %llu)\n", queue,
               (unsigned long long)tiles, rep, w[0], w[1], w[2], w[3]);
      }
      if (err != cudaSuccess || got[0] != tot) {
        ++bad;
        printf("queue=%d tiles=%llu rep=%d err=%d got=%llu want=%llu\n", queue, (unsigned long long)tiles, rep,
               (int)err, got[0], tot);
        std::vector<unsigned long long> dbg(1 << 16);
        cudaMemcpyFromSymbol(dbg.data(), g_dbg, 8 << 16);
        const uint64_t per_wave = (uint64_t)sms * 4 * 256;
        uint64_t blocks = sms * ((tiles + per_wave - 1) / per_wave);
        blocks = std::min<uint64_t>(blocks, (tiles + 31) / 32);
        uint64_t S = (tiles + blocks - 1) / blocks;
        blocks = (tiles + S - 1) / S;
        unsigned long long want = 0;
        int shown = 0;
        for (uint64_t b = 0; b < blocks; ++b) {
          if (dbg[b] != want && shown++ < 6)
            printf("  block %llu: base %llu want %llu (S=%llu)\n", (unsigned long long)b, dbg[b],
                   want, (unsigned long long)S);
          for (uint64_t t = b * S; t < (b + 1) * S && t < tiles; ++t) want += info[t];
        }
      }
    }
    cudaFree(d_info); cudaFree(d_masks); cudaFree(d_bs); cudaFree(d_cnt);
    cudaFree(d_work); cudaFree(d_dq); cudaFree(d_out);
  }
  printf("emit_unit bad=%d\n", bad);
  return bad != 0;
}
