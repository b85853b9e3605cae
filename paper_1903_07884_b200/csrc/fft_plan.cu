// Host side of the FFT engine: radix factorisation, Bluestein sizing and a
// per-device cache of twiddle / chirp tables (generated in long double on the
// host, uploaded once, never freed -- they are a few hundred KB in total).
#include <cmath>
#include <cstdarg>
#include <map>
#include <mutex>
#include <vector>

#include "fft.cuh"

namespace vx {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
  return VX_ECUDA;
}

int device_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

int device_sm_count() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}


static bool factorize(int n, std::vector<int>& out) {
  out.clear();
  int e2 = 0;
  while (n % 2 == 0) { n /= 2; ++e2; }
  while (e2 >= 3) { out.push_back(8); e2 -= 3; }
  if (e2 == 2) out.push_back(4);
  if (e2 == 1) out.push_back(2);
  for (int p : {3, 5, 7, 11, 13})
    while (n % p == 0) { n /= p; out.push_back(p); }
  return n == 1;
}

bool fft_is_smooth(int n) {
  std::vector<int> f;
  return n >= 1 && factorize(n, f);
}

int fft_good_length(int n) {
  int m = n < 1 ? 1 : n;
  while (!fft_is_smooth(m)) ++m;
  return m;
}

static int bluestein_length(int n) {
  // smallest 2^a 3^b 5^c >= 2n-1 (keeps the inner transform on fast radices)
  int target = 2 * n - 1, best = 1 << 30;
  for (long a = 1; a < (1L << 31); a *= 2)
    for (long b = a; b < (1L << 31); b *= 3)
      for (long c = b; c < (1L << 31); c *= 5) {
        if (c >= target && c < best) best = (int)c;
        if (c >= target) break;
      }
  return best;
}

struct PlanKey {
  int dev, n;
  bool operator<(const PlanKey& o) const { return dev != o.dev ? dev < o.dev : n < o.n; }
};

static std::mutex g_mu;
static std::map<PlanKey, FftPlan> g_plans;

static int upload(const std::vector<double2>& h, const double2** out) {
  double2* d = nullptr;
  VX_CUDA(cudaMalloc(&d, h.size() * sizeof(double2)));
  VX_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
  *out = d;
  return VX_OK;
}

static int upload_int(const std::vector<int>& h, const int** out) {
  int* d = nullptr;
  VX_CUDA(cudaMalloc(&d, h.size() * sizeof(int)));
  VX_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
  *out = d;
  return VX_OK;
}

static std::vector<double2> roots(int L) {
  std::vector<double2> t(L);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int m = 0; m < L; ++m) {
    long double a = two_pi * (long double)m / (long double)L;
    t[m] = make_double2((double)cosl(a), (double)-sinl(a));
  }
  return t;
}

static void host_fft(std::vector<double2>& a) {  // naive-ish O(L^2) host DFT (plan time only)
  const int L = (int)a.size();
  std::vector<double2> w = roots(L), out(L);
  for (int k = 0; k < L; ++k) {
    long double re = 0, im = 0;
    for (int j = 0; j < L; ++j) {
      const double2 t = w[(long)j * k % L];
      re += (long double)a[j].x * t.x - (long double)a[j].y * t.y;
      im += (long double)a[j].x * t.y + (long double)a[j].y * t.x;
    }
    out[k] = make_double2((double)re, (double)im);
  }
  a.swap(out);
}

int fft_get_plan(int n, FftPlan* out) {
  VX_REQUIRE(n >= 1, "FFT length must be >= 1 (got %d)", n);
  int dev = 0;
  VX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_plans.find({dev, n});
  if (it != g_plans.end()) { *out = it->second; return VX_OK; }
  FftPlan p{};
  p.n = n;
  std::vector<int> f;
  if (factorize(n, f)) {
    p.bluestein = 0;
    p.L = n;
  } else {
    p.bluestein = 1;
    p.L = bluestein_length(n);
    factorize(p.L, f);
  }
  VX_REQUIRE((int)f.size() <= FFT_MAX_STAGES, "FFT length %d needs too many stages", n);
  p.nst = (int)f.size();
  for (int i = 0; i < p.nst; ++i) p.radix[i] = f[i];
  {
    int m = p.L;
    for (int i = 0; i < p.nst; ++i) {
      m /= p.radix[i];
      p.fd_m[i] = FastDiv((unsigned)m);
      p.fd_nb[i] = FastDiv((unsigned)(p.L / p.radix[i]));
    }
  }
  int st = upload(roots(p.L), &p.tw);
  if (st) return st;
  {
    const long double two_pi = 6.283185307179586476925286766559005768L;
    p.nhi = (p.L + 63) / 64;
    std::vector<double2> hi(p.nhi), lo(64);
    for (int a = 0; a < p.nhi; ++a) {
      long double ang = two_pi * (long double)(64L * a) / (long double)p.L;
      hi[a] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
    for (int b = 0; b < 64; ++b) {
      long double ang = two_pi * (long double)b / (long double)p.L;
      lo[b] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
    if ((st = upload(hi, &p.tw_hi)) || (st = upload(lo, &p.tw_lo))) return st;
  }
  // digit-reversal maps of the DIF with this radix sequence
  std::vector<int> pos_of(p.L), k_of(p.L);
  for (int k = 0; k < p.L; ++k) {
    int rem = k, m = p.L, pos = 0;
    for (int s = 0; s < p.nst; ++s) {
      m /= p.radix[s];
      pos += (rem % p.radix[s]) * m;
      rem /= p.radix[s];
    }
    pos_of[k] = pos;
    k_of[pos] = k;
  }
  if ((st = upload_int(pos_of, &p.pos_of)) || (st = upload_int(k_of, &p.k_of))) return st;
  if (p.bluestein) {
    std::vector<double2> chirp(n);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < n; ++j) {
      long long q = ((long long)j * j) % (2LL * n);  // exact angle reduction
      long double a = pi * (long double)q / (long double)n;
      chirp[j] = make_double2((double)cosl(a), (double)-sinl(a));
    }
    std::vector<double2> b(p.L, make_double2(0, 0));
    for (int l = 0; l < n; ++l) {
      double2 c = make_double2(chirp[l].x, -chirp[l].y);
      b[l] = c;
      if (l) b[p.L - l] = c;
    }
    host_fft(b);
    std::vector<double2> brev(p.L);
    for (int pos = 0; pos < p.L; ++pos) {
      brev[pos] = b[k_of[pos]];
      brev[pos].x /= p.L;
      brev[pos].y /= p.L;
    }
    if ((st = upload(chirp, &p.chirp))) return st;
    if ((st = upload(brev, &p.bhat_rev))) return st;
    // register Bluestein: the smallest square R^2 >= 2n-1 of a register DFT length
    for (int R : {16, 20, 24, 28, 32}) {
      if (R * R < 2 * n - 1) continue;
      const int M = R * R;
      std::vector<double2> bm(M, make_double2(0, 0));
      for (int l = 0; l < n; ++l) {
        const double2 c = make_double2(chirp[l].x, -chirp[l].y);
        bm[l] = c;
        if (l) bm[M - l] = c;
      }
      host_fft(bm);
      for (auto& v : bm) { v.x /= M; v.y /= M; }
      if ((st = upload(bm, &p.blue_bhat)) || (st = upload(roots(M), &p.blue_tw))) return st;
      p.blue_R = R;
      break;
    }
  }
  g_plans[{dev, n}] = p;
  *out = p;
  return VX_OK;
}

int fft_threads_for(const FftPlan& p, int W) {
  long work = (long)W * p.L / 4;  // ~2-4 butterflies per thread per stage
  int t = (int)((work + 31) / 32 * 32);
  if (t < 64) t = 64;
  if (t > 512) t = 512;
  return t;
}

}  // namespace vx

extern "C" const char* vx_last_error(void) { return vx::g_err.c_str(); }

extern "C" int vx_version(void) { return VX_ABI_VERSION; }

extern "C" int vx_fft_good_length(int n) { return vx::fft_good_length(n); }

extern "C" int vx_fft_is_smooth(int n) { return vx::fft_is_smooth(n) ? 1 : 0; }
