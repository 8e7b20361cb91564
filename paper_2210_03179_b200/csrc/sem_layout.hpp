// sem_layout.hpp -- element-local owned-slot order (host + device).
//
// Element e owns the nodes with local indices (a+1, b+1, c+1), a,b,c in [0,N).
// Inside the element block the owned slots are ordered INTERIOR-FIRST:
//   [0, (N-1)^3)                 nodes with a,b,c < N-1 (single contributor,
//                                finished by the element kernel K1), x fastest
//   [(N-1)^3, N^3)               "shared" nodes (some index == N-1, i.e. local N),
//                                lexicographic (c, b, a) -- finished by K2
//   [N^3, NOS)                   zero pad so every element block is 16-byte aligned
// so K1's interior epilogue and K2 both touch one contiguous range per element
// (coalesced, TMA-bulk-copyable) instead of scattered 56-byte rows.
#pragma once

#ifdef __CUDACC__
#define CMG_HD __host__ __device__ __forceinline__
#else
#define CMG_HD inline
#endif

namespace cmg {

CMG_HD constexpr int sem_nos(int N) { return (N * N * N + 1) & ~1; }          // slots per element
CMG_HD constexpr int sem_nint(int N) { return (N - 1) * (N - 1) * (N - 1); }  // interior slots
CMG_HD constexpr int sem_nshared(int N) { return N * N * N - (N - 1) * (N - 1) * (N - 1); }

// rank of a shared node among the element's shared nodes, lexicographic (c, b, a)
CMG_HD int sem_shared_rank(int N, int a, int b, int c) {
  if (c == N - 1) return (N - 1) * (2 * N - 1) + b * N + a;
  const int base = c * (2 * N - 1);
  if (b == N - 1) return base + (N - 1) + a;
  return base + b;  // a == N-1
}

// element-local slot position of owned node (a, b, c)
CMG_HD int sem_pos(int N, int a, int b, int c) {
  if (a < N - 1 && b < N - 1 && c < N - 1) return a + (N - 1) * (b + (N - 1) * c);
  return sem_nint(N) + sem_shared_rank(N, a, b, c);
}

// inverse of the shared rank
CMG_HD void sem_shared_abc(int N, int s, int& a, int& b, int& c) {
  const int P = (N - 1) * (2 * N - 1);
  if (s >= P) {
    const int t = s - P;
    c = N - 1;
    b = t / N;
    a = t - b * N;
  } else {
    c = s / (2 * N - 1);
    const int t = s - c * (2 * N - 1);
    if (t < N - 1) {
      b = t;
      a = N - 1;
    } else {
      b = N - 1;
      a = t - (N - 1);
    }
  }
}

// inverse of sem_pos; returns false for pad slots
CMG_HD bool sem_abc(int N, int p, int& a, int& b, int& c) {
  const int ni = sem_nint(N);
  if (p < ni) {
    a = p % (N - 1);
    b = (p / (N - 1)) % (N - 1);
    c = p / ((N - 1) * (N - 1));
    return true;
  }
  if (p >= N * N * N) return false;
  sem_shared_abc(N, p - ni, a, b, c);
  return true;
}

}  // namespace cmg
