// TEST INFRASTRUCTURE — the CPU baseline harness (bench.py's cpu_baseline leg
// and `bench.py --impl reference`). It links the *compiled reference*
// (oracle/_ref/libgte_ref.a) and times the reference's own per-head
// sparse_attention + sparse_attention_backward (proj/src/attention.cpp:96,241)
// on a pattern read from a binary CSR file, head-parallel on T host threads
// (the reference is pure and reentrant), as SURVEY.md §8(d4)(ii)
// prescribes. A bounded sample is taken by keeping the first R rows of the
// pattern and emptying the rest (empty rows are skipped by the reference).
//
// With more host threads than heads, each head's rows are also cut into
// `chunks` contiguous ranges: every (head, chunk) work item calls the
// reference on the sub-pattern of its rows (other rows empty), and the
// chunks' dK/dV partial sums are added afterwards, inside the timed region.
//
// usage: ref_cpu_bench <csr.bin> <heads> <dh> <threads> <sample_rows> <steps> <warmup> <seed> [chunks]
// csr.bin: int64 n, int64 nnz, int64 row_off[n+1], int64 cols[nnz] (little endian)
// prints one JSON line: {"step_s":[...], "rows":R, "threads":T, ...}
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <span>
#include <thread>
#include <vector>

#include "gte/attention.hpp"

using namespace gte;

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: %s csr.bin heads dh threads sample_rows steps warmup seed\n", argv[0]);
    return 2;
  }
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) {
    std::fprintf(stderr, "cannot open %s\n", argv[1]);
    return 2;
  }
  int64_t n = 0, nnz = 0;
  if (std::fread(&n, 8, 1, f) != 1 || std::fread(&nnz, 8, 1, f) != 1) return 2;
  std::vector<Index> off(static_cast<size_t>(n + 1)), cols(static_cast<size_t>(nnz));
  if (std::fread(off.data(), 8, off.size(), f) != off.size()) return 2;
  if (std::fread(cols.data(), 8, cols.size(), f) != cols.size()) return 2;
  std::fclose(f);
  const int H = std::atoi(argv[2]), dh = std::atoi(argv[3]);
  int T = std::atoi(argv[4]);
  int64_t R = std::atoll(argv[5]);
  const int steps = std::atoi(argv[6]), warmup = std::atoi(argv[7]);
  const uint64_t seed = std::strtoull(argv[8], nullptr, 10);
  if (R <= 0 || R > n) R = n;
  if (T < 1) T = 1;
  int C = argc > 9 ? std::atoi(argv[9]) : 1;
  if (C < 1) C = 1;

  // Sampled pattern: rows [0, R) keep their pairs, the rest attend nothing.
  AttnPattern pat;
  pat.rows = n;
  pat.row_offsets.assign(static_cast<size_t>(n + 1), 0);
  for (int64_t i = 0; i <= n; ++i) pat.row_offsets[static_cast<size_t>(i)] = off[static_cast<size_t>(i < R ? i : R)];
  pat.cols.assign(cols.begin(), cols.begin() + off[static_cast<size_t>(R)]);
  const int64_t e_s = pat.nnz();
  // row chunks: near-equal pair counts per chunk
  std::vector<AttnPattern> parts(static_cast<size_t>(C));
  std::vector<int64_t> ebeg(static_cast<size_t>(C) + 1, 0);
  {
    int64_t r0 = 0;
    for (int c = 0; c < C; ++c) {
      int64_t r1 = r0;
      const int64_t target = e_s * (c + 1) / C;
      while (r1 < R && (c == C - 1 || off[static_cast<size_t>(r1)] < target)) ++r1;
      if (c == C - 1) r1 = R;
      AttnPattern& p = parts[static_cast<size_t>(c)];
      p.rows = n;
      p.row_offsets.assign(static_cast<size_t>(n + 1), 0);
      const int64_t b = off[static_cast<size_t>(r0)];
      for (int64_t i = 0; i <= n; ++i) {
        const int64_t ii = i < r0 ? r0 : (i < r1 ? i : r1);
        p.row_offsets[static_cast<size_t>(i)] = off[static_cast<size_t>(ii)] - b;
      }
      p.cols.assign(cols.begin() + b, cols.begin() + off[static_cast<size_t>(r1)]);
      ebeg[static_cast<size_t>(c)] = b;
      r0 = r1;
    }
    ebeg[static_cast<size_t>(C)] = e_s;
  }

  std::mt19937_64 rng(seed);
  std::vector<Matrix> q, k, v, up;
  for (int h = 0; h < H; ++h) {
    q.push_back(Matrix::randn(n, dh, 1.0, rng));
    k.push_back(Matrix::randn(n, dh, 1.0, rng));
    v.push_back(Matrix::randn(n, dh, 1.0, rng));
    up.push_back(Matrix::randn(n, dh, 1.0, rng));
  }
  std::vector<Real> bias(static_cast<size_t>(e_s));
  std::normal_distribution<Real> nd(0.0, 0.3);
  for (Real& b : bias) b = nd(rng);

  std::vector<double> times;
  volatile double sink = 0;
  for (int s = 0; s < warmup + steps; ++s) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    std::vector<double> partial(static_cast<size_t>(T), 0.0);
    const int items = H * C;
    std::vector<AttnGrads> grads(static_cast<size_t>(items));
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        for (int it = t; it < items; it += T) {
          const int h = it / C, c = it % C;
          const AttnPattern& p = C == 1 ? pat : parts[static_cast<size_t>(c)];
          std::span<const Real> b(bias.data() + ebeg[static_cast<size_t>(c)],
                                  static_cast<size_t>(ebeg[static_cast<size_t>(c) + 1] - ebeg[static_cast<size_t>(c)]));
          auto r = sparse_attention(q[h], k[h], v[h], p, b);
          grads[static_cast<size_t>(it)] = sparse_attention_backward(q[h], k[h], v[h], p, b, {}, up[h]);
          partial[static_cast<size_t>(t)] += r.output(0, 0) + grads[static_cast<size_t>(it)].dq(0, 0);
        }
      });
    }
    for (auto& th : pool) th.join();
    pool.clear();
    if (C > 1) {  // sum the chunks' dK/dV partials per head (column scatter of the backward)
      for (int t = 0; t < T && t < H; ++t) {
        pool.emplace_back([&, t] {
          for (int h = t; h < H; h += T) {
            AttnGrads& g0 = grads[static_cast<size_t>(h * C)];
            for (int c = 1; c < C; ++c) {
              const AttnGrads& gc = grads[static_cast<size_t>(h * C + c)];
              for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < dh; ++j) {
                  g0.dk(i, j) += gc.dk(i, j);
                  g0.dv(i, j) += gc.dv(i, j);
                }
            }
            partial[static_cast<size_t>(t)] += g0.dk(0, 0);
          }
        });
      }
    }
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    for (double p : partial) sink = sink + p;
    if (s >= warmup) times.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  std::printf("{\"rows\": %lld, \"pairs\": %lld, \"threads\": %d, \"chunks\": %d, \"heads\": %d, \"dh\": %d, \"step_s\": [",
              static_cast<long long>(R), static_cast<long long>(e_s), T, C, H, dh);
  for (size_t i = 0; i < times.size(); ++i) std::printf("%s%.6f", i ? ", " : "", times[i]);
  std::printf("]}\n");
  return sink == 12345.678 ? 1 : 0;
}
