// hadacodec-b200: the reference's geometric path tracer on the GPU —
// the real caller of the shading channel loops:
//   render                   renderer.cpp:437-612, :624-628
//   render_latent_multipass  renderer.cpp:630-659 (k/3 three-channel passes, slice_pass :274-283)
//   compile_scene            renderer.cpp:117-272 (per-mode albedo / emission / luma rows)
//
// Same algorithm, same numbers: geometry in fp64, per-sample channel arithmetic in fp32,
// per-pixel fp64 accumulation over samples in sample order, the per-(pixel, sample, lane)
// xoshiro256++ streams of Rng::pixel_stream (rng.cpp:45-55).  The file is compiled with
// -fmad=false (build.py) so every expression rounds exactly like the reference's x86-64
// build (no contraction); sqrt and the divisions are IEEE on both sides, and the one
// libm call on the path, cos / sin of the continuation direction, is evaluated correctly
// rounded (sincos_cr), i.e. as glibc returns it.
//
// One thread renders one pixel (all its samples), like a reference worker; channel
// vectors are compile-time sized (C = 3, 6, 9 registers; C = n spectral in local
// memory).  Scene tables (albedo, emission, luma) are small device arrays read through
// the read-only path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hadacodec_b200.h"
#include "hc_internal.h"

namespace hcb {
namespace {

constexpr double kRayEpsilon = 1e-4;
constexpr double kPi = 3.14159265358979323846;

// ---------------------------------------------------------------- fp64 vector helpers
struct V3 {
  double x, y, z;
};
__host__ __device__ inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__host__ __device__ inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__host__ __device__ inline V3 mul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__host__ __device__ inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__host__ __device__ inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__host__ __device__ inline V3 normalize(V3 a) {  // renderer.cpp:41-45 (callers guarantee len > 0)
  const double len = sqrt(dot(a, a));
  return mul(a, 1.0 / len);
}
inline V3 v3(const double* p) { return {p[0], p[1], p[2]}; }

struct Ray {
  V3 o, d;
};

struct Wall {  // renderer.cpp:84-90
  int axis;
  double plane, lo0, hi0, lo1, hi1;
  V3 n;
  int material;
};
struct Object {  // renderer.hpp:32-39
  int kind;  // 0 sphere, 1 block
  V3 center;
  double radius;
  V3 bmin, bmax;
  int material;
};
struct LightG {  // renderer.cpp:79-82
  V3 corner, eu, ev, n;
  double area;
};

struct Frame {  // renderer.cpp:52-55
  V3 origin, right, up, forward;
  double tan_half, aspect;
};

struct RenderParams {
  Frame cam;
  Wall walls[6];
  const Object* objects;
  int n_objects;
  const LightG* lights;
  int n_lights;
  const float* albedo;    // n_materials x C
  const float* emission;  // n_lights x C
  const float* luma;      // C
  int width, height, spp, max_depth;
  uint64_t seed;
  uint64_t eval_unit;
  float* image;            // H x W x C
  uint64_t* hashes;        // H x W or null
  unsigned long long* evals;
};

// ---------------------------------------------------------------- RNG (rng.cpp:7-81)
__device__ inline uint64_t splitmix64_next(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
struct Rng {
  uint64_t s[4];
  __device__ explicit Rng(uint64_t seed) {
    uint64_t st = seed;
    for (int i = 0; i < 4; ++i) s[i] = splitmix64_next(st);
  }
  // Rng::pixel_stream (rng.cpp:45-55)
  __device__ static Rng pixel(uint64_t seed, int x, int y, int sample, uint32_t lane) {
    uint64_t st = seed;
    uint64_t h = splitmix64_next(st);
    st = h ^ (static_cast<uint64_t>(static_cast<uint32_t>(x)) | (static_cast<uint64_t>(static_cast<uint32_t>(y)) << 32));
    h = splitmix64_next(st);
    st = h ^ (static_cast<uint64_t>(static_cast<uint32_t>(sample)) | (static_cast<uint64_t>(lane) << 32));
    return Rng(splitmix64_next(st));
  }
  __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  __device__ uint64_t next() {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  __device__ double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  __device__ uint32_t index(uint32_t n) { return static_cast<uint32_t>(next() % n); }
};

__device__ inline uint64_t fnv_bytes(uint64_t h, const void* p, int size) {  // fnv1a64 (rng.cpp:7-15)
  const unsigned char* b = static_cast<const unsigned char*>(p);
  for (int i = 0; i < size; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// ---------------------------------------------------------------- correctly rounded sin / cos
// The continuation direction uses cos(phi) and sin(phi) (renderer.cpp:521-525).  CUDA's
// fp64 sin / cos are within 2 ulp, glibc's are (almost always) correctly rounded; a 1-ulp
// difference changes nothing in the image but does change the exact hit points that the
// per-pixel path hashes (FNV of the hit positions' bits) fold in.  So phi in [0, 2 pi) is
// reduced with a 3-part pi/2 (exact multiples), sin / cos of the reduced argument are
// evaluated in double-double (Taylor to 1/29!, error < 1e-31) and rounded once: the
// correctly rounded result, i.e. glibc's.
struct DD {
  double hi, lo;
};
__device__ inline DD two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ inline DD quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ inline DD dd_add(DD a, DD b) {
  const DD s = two_sum(a.hi, b.hi);
  return quick_two_sum(s.hi, s.lo + (a.lo + b.lo));
}
__device__ inline DD dd_mul(DD a, DD b) {
  const double p = a.hi * b.hi;
  const double e = fma(a.hi, b.hi, -p);
  return quick_two_sum(p, e + (a.hi * b.lo + a.lo * b.hi));
}
__constant__ double kInvFact[30][2] = {
    {1.0, 0.0},
    {1.0, 0.0},
    {0.5, 0.0},
    {0.16666666666666666, 9.25185853854297e-18},
    {0.041666666666666664, 2.3129646346357427e-18},
    {0.008333333333333333, 1.1564823173178714e-19},
    {0.001388888888888889, -5.300543954373577e-20},
    {0.0001984126984126984, 1.7209558293420705e-22},
    {2.48015873015873e-05, 2.1511947866775882e-23},
    {2.7557319223985893e-06, -1.858393274046472e-22},
    {2.755731922398589e-07, 2.3767714622250297e-23},
    {2.505210838544172e-08, -1.448814070935912e-24},
    {2.08767569878681e-09, -1.20734505911326e-25},
    {1.6059043836821613e-10, 1.2585294588752098e-26},
    {1.1470745597729725e-11, 2.0655512752830745e-28},
    {7.647163731819816e-13, 7.03872877733453e-30},
    {4.779477332387385e-14, 4.399205485834081e-31},
    {2.8114572543455206e-15, 1.6508842730861433e-31},
    {1.5619206968586225e-16, 1.1910679660273754e-32},
    {8.22063524662433e-18, 2.2141894119604265e-34},
    {4.110317623312165e-19, 1.4412973378659527e-36},
    {1.9572941063391263e-20, -1.3643503830087908e-36},
    {8.896791392450574e-22, -7.911402614872376e-38},
    {3.868170170630684e-23, -8.843177655482344e-40},
    {1.6117375710961184e-24, -3.6846573564509766e-41},
    {6.446950284384474e-26, -1.9330404233703465e-42},
    {2.4795962632247976e-27, -1.2953730964765229e-43},
    {9.183689863795546e-29, 1.4303150396787322e-45},
    {3.279889237069838e-30, 1.5117542744029879e-46},
    {1.1309962886447716e-31, 1.0498015412959506e-47}
};

__device__ inline void sincos_cr(double x, double* sn, double* cs) {
  const double P1 = 1.57079632673412561417e+00, P2 = 6.07710050630396597660e-11,
               P3 = 2.02226624871116645580e-21, P3T = 8.47842766036889956997e-32;
  const int k = static_cast<int>(rint(x * 0.63661977236758134308));
  const double kd = static_cast<double>(k);
  DD r = two_sum(x, -kd * P1);
  r = dd_add(r, {-kd * P2, 0.0});
  r = dd_add(r, {-kd * P3, 0.0});
  r = dd_add(r, {-kd * P3T, 0.0});
  const DD r2 = dd_mul(r, r);
  // sin r = r (1 - r^2/3! + r^4/5! - ...), cos r = 1 - r^2/2! + r^4/4! - ...
  DD ps = {kInvFact[29][0], kInvFact[29][1]}, pc = {kInvFact[28][0], kInvFact[28][1]};
  for (int j = 27; j >= 1; j -= 2) {  // ps over odd factorials 29, 27, ..., 3, 1
    ps = dd_mul(ps, {-r2.hi, -r2.lo});
    ps = dd_add(ps, {kInvFact[j][0], kInvFact[j][1]});
  }
  for (int j = 26; j >= 0; j -= 2) {  // pc over even factorials 28, 26, ..., 2, 0
    pc = dd_mul(pc, {-r2.hi, -r2.lo});
    pc = dd_add(pc, {kInvFact[j][0], kInvFact[j][1]});
  }
  const DD s = dd_mul(ps, r);
  const double sr = s.hi + s.lo, cr = pc.hi + pc.lo;
  switch (k & 3) {
    case 0: *sn = sr; *cs = cr; break;
    case 1: *sn = cr; *cs = -sr; break;
    case 2: *sn = -sr; *cs = -cr; break;
    default: *sn = -cr; *cs = sr; break;
  }
}

// ---------------------------------------------------------------- intersection (renderer.cpp:274-432)
struct Hit {
  double t;
  V3 p, n;
  int prim, material, light;
};

__device__ inline bool hit_wall(const Wall& w, const Ray& ray, double t_min, double t_max, Hit* hit) {
  if (w.material < 0) return false;
  const double o = w.axis == 0 ? ray.o.x : (w.axis == 1 ? ray.o.y : ray.o.z);
  const double d = w.axis == 0 ? ray.d.x : (w.axis == 1 ? ray.d.y : ray.d.z);
  if (fabs(d) < 1e-12) return false;
  const double t = (w.plane - o) / d;
  if (t <= t_min || t >= t_max || t >= hit->t) return false;
  const V3 p = add(ray.o, mul(ray.d, t));
  const double u = w.axis == 0 ? p.y : p.x;
  const double v = w.axis == 2 ? p.y : p.z;
  if (u < w.lo0 || u > w.hi0 || v < w.lo1 || v > w.hi1) return false;
  hit->t = t;
  hit->p = p;
  hit->n = w.n;
  hit->material = w.material;
  hit->light = -1;
  return true;
}

__device__ inline bool hit_sphere(const Object& s, const Ray& ray, double t_min, double t_max, Hit* hit) {
  const V3 oc = sub(ray.o, s.center);
  const double b = dot(oc, ray.d);
  const double c = dot(oc, oc) - s.radius * s.radius;
  const double disc = b * b - c;
  if (disc < 0.0) return false;
  const double sq = sqrt(disc);
  double t = -b - sq;
  if (t <= t_min) t = -b + sq;
  if (t <= t_min || t >= t_max || t >= hit->t) return false;
  hit->t = t;
  hit->p = add(ray.o, mul(ray.d, t));
  hit->n = mul(sub(hit->p, s.center), 1.0 / s.radius);
  hit->material = s.material;
  hit->light = -1;
  return true;
}

__device__ inline bool hit_block(const Object& blk, const Ray& ray, double t_min, double t_max, Hit* hit) {
  double t0 = t_min, t1 = t_max < hit->t ? t_max : hit->t;
  int axis_near = -1;
  const double o[3] = {ray.o.x, ray.o.y, ray.o.z};
  const double d[3] = {ray.d.x, ray.d.y, ray.d.z};
  const double lo[3] = {blk.bmin.x, blk.bmin.y, blk.bmin.z};
  const double hi[3] = {blk.bmax.x, blk.bmax.y, blk.bmax.z};
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0) {
      if (o[a] < lo[a] || o[a] > hi[a]) return false;
      continue;
    }
    const double inv = 1.0 / d[a];
    double ta = (lo[a] - o[a]) * inv;
    double tb = (hi[a] - o[a]) * inv;
    if (ta > tb) {
      const double tmp = ta;
      ta = tb;
      tb = tmp;
    }
    if (ta > t0) {
      t0 = ta;
      axis_near = a;
    }
    t1 = tb < t1 ? tb : t1;
    if (t0 >= t1) return false;
  }
  if (axis_near < 0) return false;  // origin inside: treat as miss
  hit->t = t0;
  hit->p = add(ray.o, mul(ray.d, t0));
  V3 n{0, 0, 0};
  const double sign = d[axis_near] > 0.0 ? -1.0 : 1.0;
  if (axis_near == 0) n.x = sign;
  if (axis_near == 1) n.y = sign;
  if (axis_near == 2) n.z = sign;
  hit->n = n;
  hit->material = blk.material;
  hit->light = -1;
  return true;
}

__device__ inline bool hit_light(const LightG& l, const Ray& ray, double t_min, double t_max, Hit* hit) {
  const double denom = dot(ray.d, l.n);
  if (fabs(denom) < 1e-12) return false;
  const double t = dot(sub(l.corner, ray.o), l.n) / denom;
  if (t <= t_min || t >= t_max || t >= hit->t) return false;
  const V3 q = sub(add(ray.o, mul(ray.d, t)), l.corner);
  const double uu = dot(l.eu, l.eu), uv = dot(l.eu, l.ev), vv = dot(l.ev, l.ev);
  const double qu = dot(q, l.eu), qv = dot(q, l.ev);
  const double det = uu * vv - uv * uv;
  const double u = (vv * qu - uv * qv) / det;
  const double v = (uu * qv - uv * qu) / det;
  if (u < 0.0 || u > 1.0 || v < 0.0 || v > 1.0) return false;
  hit->t = t;
  hit->p = add(ray.o, mul(ray.d, t));
  hit->n = l.n;
  hit->material = -1;
  return true;
}

// Primitive ids: walls 0..5, objects, lights (renderer.cpp:412-432).
__device__ inline bool intersect(const RenderParams& p, const Ray& ray, double t_min, double t_max, Hit* hit) {
  hit->t = INFINITY;
  hit->prim = -1;
  for (int w = 0; w < 6; ++w)
    if (hit_wall(p.walls[w], ray, t_min, t_max, hit)) hit->prim = w;
  for (int i = 0; i < p.n_objects; ++i) {
    const Object obj = p.objects[i];
    const bool got = obj.kind == 0 ? hit_sphere(obj, ray, t_min, t_max, hit) : hit_block(obj, ray, t_min, t_max, hit);
    if (got) hit->prim = 6 + i;
  }
  for (int i = 0; i < p.n_lights; ++i) {
    if (hit_light(p.lights[i], ray, t_min, t_max, hit)) {
      hit->prim = 6 + p.n_objects + i;
      hit->light = i;
    }
  }
  return hit->prim >= 0;
}

// ---------------------------------------------------------------- path kernel (renderer.cpp:448-563)
// One sample of one pixel (renderer.cpp:456-559): radiance rad[C]; shading units added to
// *evals; the hit sequence folded into *hash when hash != nullptr.
template <int C>
__device__ __forceinline__ void trace_sample(const RenderParams& p, int x, int y, int s, float* rad,
                                             unsigned long long* evals, uint64_t* hash) {
  float thr[C];
  const int nl = p.n_lights;
  Rng geo = Rng::pixel(p.seed, x, y, s, 0);
  Rng rr = Rng::pixel(p.seed, x, y, s, 1);
  const double jx = geo.uniform();
  const double jy = geo.uniform();
  Ray ray;
  {  // camera_ray (renderer.cpp:63-68)
    const double px = x + jx, py = y + jy;
    const double u = (2.0 * px / p.width - 1.0) * p.cam.tan_half * p.cam.aspect;
    const double v = (1.0 - 2.0 * py / p.height) * p.cam.tan_half;
    ray = {p.cam.origin, normalize(add(add(p.cam.forward, mul(p.cam.right, u)), mul(p.cam.up, v)))};
  }
  for (int c = 0; c < C; ++c) {
    thr[c] = 1.0f;
    rad[c] = 0.0f;
  }
  for (int depth = 0;; ++depth) {
    Hit hit;
    if (!intersect(p, ray, kRayEpsilon, INFINITY, &hit)) break;
    if (hash) {  // hash_hit (renderer.cpp:436-442)
      *hash = fnv_bytes(*hash, &hit.p.x, 8);
      *hash = fnv_bytes(*hash, &hit.p.y, 8);
      *hash = fnv_bytes(*hash, &hit.p.z, 8);
      const uint32_t prim = static_cast<uint32_t>(hit.prim);
      *hash = fnv_bytes(*hash, &prim, 4);
    }
    if (hit.light >= 0) {  // emitters seen directly by the camera only
      if (depth == 0 && dot(ray.d, hit.n) < 0.0) {
        const float* le = p.emission + hit.light * C;
        for (int c = 0; c < C; ++c) rad[c] += thr[c] * __ldg(le + c);
      }
      break;
    }
    if (p.max_depth >= 0 && depth >= p.max_depth) break;
    *evals += p.eval_unit;
    const V3 n_sh = dot(hit.n, ray.d) < 0.0 ? hit.n : mul(hit.n, -1.0);
    const float* albedo = p.albedo + hit.material * C;

    if (nl > 0) {  // next-event estimation: one area sample on one light
      const uint32_t li = geo.index(static_cast<uint32_t>(nl));
      const double lu = geo.uniform();
      const double lv = geo.uniform();
      const LightG lg = p.lights[li];
      const V3 lp = add(add(lg.corner, mul(lg.eu, lu)), mul(lg.ev, lv));
      const V3 d = sub(lp, hit.p);
      const double dist2 = dot(d, d);
      const double dist = sqrt(dist2);
      if (dist > kRayEpsilon) {
        const V3 wi = mul(d, 1.0 / dist);
        const double cos_s = dot(n_sh, wi);
        const double cos_l = -dot(lg.n, wi);
        if (cos_s > 0.0 && cos_l > 0.0) {
          Hit occ;
          if (!intersect(p, {hit.p, wi}, kRayEpsilon, dist - kRayEpsilon, &occ)) {
            const double geom = cos_s * cos_l / dist2 * lg.area * static_cast<double>(nl) / kPi;
            const float w = static_cast<float>(geom);
            const float* le = p.emission + li * C;
            for (int c = 0; c < C; ++c) rad[c] += thr[c] * __ldg(albedo + c) * __ldg(le + c) * w;
          }
        }
      }
    }
    if (p.max_depth >= 0 && depth + 1 >= p.max_depth) break;

    // cosine-weighted continuation; throughput picks up the bare albedo
    const double u1 = geo.uniform();
    const double u2 = geo.uniform();
    const double r = sqrt(u1);
    const double phi = 2.0 * kPi * u2;
    const V3 tangent = fabs(n_sh.x) > 0.9 ? normalize(cross({0, 1, 0}, n_sh)) : normalize(cross({1, 0, 0}, n_sh));
    const V3 bitangent = cross(n_sh, tangent);
    const double om = 1.0 - u1;
    double sin_phi, cos_phi;
    sincos_cr(phi, &sin_phi, &cos_phi);
    const V3 dir = normalize(add(add(mul(tangent, r * cos_phi), mul(bitangent, r * sin_phi)),
                                 mul(n_sh, sqrt(om > 0.0 ? om : 0.0))));
    for (int c = 0; c < C; ++c) thr[c] *= __ldg(albedo + c);

    if (p.max_depth < 0 && depth >= 5) {  // Russian roulette on throughput luminance
      float acc = 0.0f;
      for (int c = 0; c < C; ++c) acc += __ldg(p.luma + c) * thr[c];
      const float q = acc < 0.05f ? 0.05f : (acc > 1.0f ? 1.0f : acc);
      if (rr.uniform() >= static_cast<double>(q)) break;
      const float inv_q = 1.0f / q;
      for (int c = 0; c < C; ++c) thr[c] *= inv_q;
    }
    ray = {hit.p, dir};
  }
}

// Pixel-serial form: one thread per pixel loops over its samples, like a reference
// worker (needed when path hashes are collected: the hash chains the hits of all samples
// in order).
template <int C>
__global__ void __launch_bounds__(128) render_kernel(const __grid_constant__ RenderParams p) {
  const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (pix >= static_cast<int64_t>(p.width) * p.height) return;
  const int x = static_cast<int>(pix % p.width), y = static_cast<int>(pix / p.width);
  float rad[C];
  double accum[C];
  for (int c = 0; c < C; ++c) accum[c] = 0.0;
  uint64_t pixel_hash = 0xcbf29ce484222325ull;
  unsigned long long evals = 0;
  for (int s = 0; s < p.spp; ++s) {
    trace_sample<C>(p, x, y, s, rad, &evals, p.hashes ? &pixel_hash : nullptr);
    for (int c = 0; c < C; ++c) accum[c] += static_cast<double>(rad[c]);
  }
  const double inv_spp = 1.0 / p.spp;
  float* out = p.image + pix * C;
  for (int c = 0; c < C; ++c) out[c] = static_cast<float>(accum[c] * inv_spp);
  if (p.hashes) p.hashes[pix] = pixel_hash;
  if (evals) atomicAdd(p.evals, evals);
}

// Sample-parallel form: one thread per (sample, pixel) of a chunk of samples writes its
// radiance; accumulate_kernel then adds the chunk's samples to the per-pixel fp64 sums in
// sample order, so the image is bit-identical to the pixel-serial form with spp x the
// parallelism.
template <int C>
__global__ void __launch_bounds__(128) render_samples_kernel(const __grid_constant__ RenderParams p, int s0, int ns,
                                                             float* __restrict__ samples) {
  const int64_t P = static_cast<int64_t>(p.width) * p.height;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long evals = 0;
  if (t < P * ns) {
    const int64_t pix = t % P;
    const int j = static_cast<int>(t / P);
    const int x = static_cast<int>(pix % p.width), y = static_cast<int>(pix / p.width);
    float rad[C];
    trace_sample<C>(p, x, y, s0 + j, rad, &evals, nullptr);
    float* out = samples + (static_cast<int64_t>(j) * P + pix) * C;
    for (int c = 0; c < C; ++c) out[c] = rad[c];
  }
  // one atomic per warp
  for (int o = 16; o > 0; o >>= 1) evals += __shfl_xor_sync(0xffffffffu, evals, o);
  if ((threadIdx.x & 31) == 0 && evals) atomicAdd(p.evals, evals);
}

template <int C>
__global__ void accumulate_kernel(const float* __restrict__ samples, int64_t P, int ns, double* __restrict__ accum) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P * C; i += int64_t(gridDim.x) * blockDim.x) {
    double a = accum[i];
    for (int j = 0; j < ns; ++j) a += static_cast<double>(samples[j * P * C + i]);
    accum[i] = a;
  }
}

__global__ void finalize_kernel(const double* __restrict__ accum, int64_t count, double inv_spp,
                                float* __restrict__ image) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    image[i] = static_cast<float>(accum[i] * inv_spp);
}

// ---------------------------------------------------------------- compile_scene (renderer.cpp:201-272)
constexpr double kXyzToRgbH[9] = {3.2404542, -1.5371385, -0.4985314, -0.9692660, 1.8760108,
                                  0.0415560, 0.0556434,  -0.2040259, 1.0572252};

struct Compiled {
  int channels = 0;
  uint64_t eval_unit = 0;
  std::vector<float> luma, albedo, emission;  // flattened
  std::vector<Object> objects;
  std::vector<LightG> lights;
  Wall walls[6];
  Frame frame;
};

void fail(const char* msg) { throw std::invalid_argument(msg); }

V3 normalize_h(V3 a) {
  const double len = std::sqrt(dot(a, a));
  if (len <= 0.0) fail("renderer: zero-length vector");
  return mul(a, 1.0 / len);
}

Compiled compile_scene(hc_codec c, const hc_scene* sc, int mode, const double* d65) {
  const int n = c->n;
  Compiled cs;
  if (sc->n_materials < 0 || sc->n_objects < 0 || sc->n_lights < 0) fail("renderer: negative scene counts");
  if (sc->n_materials > 0 && !sc->materials) fail("renderer: null materials");
  for (int w = 0; w < 6; ++w)
    if (sc->wall_material[w] >= sc->n_materials) fail("renderer: wall references missing material");
  for (int i = 0; i < sc->n_objects; ++i)
    if (sc->objects[i].material < 0 || sc->objects[i].material >= sc->n_materials)
      fail("renderer: object references missing material");
  const int k = c->k;
  switch (mode) {
    case HC_RENDER_SPECTRAL: cs.channels = n; cs.eval_unit = static_cast<uint64_t>(n); break;
    case HC_RENDER_LATENT: cs.channels = k; cs.eval_unit = static_cast<uint64_t>(k / 3); break;
    case HC_RENDER_RGB: cs.channels = 3; cs.eval_unit = 1; break;
    default: fail("renderer: unknown render mode");
  }
  if (mode == HC_RENDER_RGB && !d65) fail("renderer: rgb mode needs the grid's D65 row");
  const double* xb = c->cmf.data();
  const double* yb = c->cmf.data() + n;
  const double* zb = c->cmf.data() + 2 * n;
  auto encode_d = [&](const double* s, int j) {  // encode (codec.cpp:36-46) in fp64
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += c->Ed[static_cast<size_t>(j) * n + i] * s[i];
    return acc;
  };
  // materials (renderer.cpp:230-243)
  for (int m = 0; m < sc->n_materials; ++m) {
    const double* r = sc->materials + static_cast<size_t>(m) * n;
    if (mode == HC_RENDER_SPECTRAL) {
      for (int i = 0; i < n; ++i) cs.albedo.push_back(static_cast<float>(r[i] * 1.0));
    } else if (mode == HC_RENDER_LATENT) {
      for (int j = 0; j < k; ++j) cs.albedo.push_back(static_cast<float>(encode_d(r, j) * 1.0));
    } else {  // reflectance_to_rgb (renderer.cpp:127-137): D65-weighted rows, Y of unit reflectance = 100
      double norm = 0.0;
      for (int i = 0; i < n; ++i) norm += yb[i] * d65[i];
      const double scale = 100.0 / norm;
      double xyz[3] = {0, 0, 0};
      for (int i = 0; i < n; ++i) {
        xyz[0] += scale * xb[i] * d65[i] * r[i];
        xyz[1] += scale * yb[i] * d65[i] * r[i];
        xyz[2] += scale * zb[i] * d65[i] * r[i];
      }
      for (int q = 0; q < 3; ++q) xyz[q] /= 100.0;
      for (int q = 0; q < 3; ++q) {
        const double v = kXyzToRgbH[3 * q] * xyz[0] + kXyzToRgbH[3 * q + 1] * xyz[1] + kXyzToRgbH[3 * q + 2] * xyz[2];
        cs.albedo.push_back(static_cast<float>(v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v)));
      }
    }
  }
  // lights (renderer.cpp:244-268)
  for (int l = 0; l < sc->n_lights; ++l) {
    const hc_scene_light& L = sc->lights[l];
    if (!L.spd) fail("renderer: null light spd");
    if (mode == HC_RENDER_SPECTRAL) {
      for (int i = 0; i < n; ++i) cs.emission.push_back(static_cast<float>(L.spd[i] * L.scale));
    } else if (mode == HC_RENDER_LATENT) {
      for (int j = 0; j < k; ++j) cs.emission.push_back(static_cast<float>(encode_d(L.spd, j) * L.scale));
    } else {  // emission_to_rgb (renderer.cpp:139-147)
      double x = 0, y = 0, z = 0;
      for (int i = 0; i < n; ++i) {
        x += xb[i] * L.spd[i];
        y += yb[i] * L.spd[i];
        z += zb[i] * L.spd[i];
      }
      const double xyz[3] = {x * c->dlambda, y * c->dlambda, z * c->dlambda};
      for (int q = 0; q < 3; ++q) {
        const double v = kXyzToRgbH[3 * q] * xyz[0] + kXyzToRgbH[3 * q + 1] * xyz[1] + kXyzToRgbH[3 * q + 2] * xyz[2];
        cs.emission.push_back(static_cast<float>((v > 0.0 ? v : 0.0) * L.scale));
      }
    }
    LightG g;
    g.corner = v3(L.corner);
    g.eu = v3(L.edge_u);
    g.ev = v3(L.edge_v);
    const V3 cr = cross(g.eu, g.ev);
    g.area = std::sqrt(dot(cr, cr));
    if (g.area <= 0.0) fail("renderer: degenerate light parallelogram");
    g.n = mul(cr, 1.0 / g.area);
    cs.lights.push_back(g);
  }
  // luma row (renderer.cpp:249-263, normalised so luma(ones) = 1)
  cs.luma.assign(static_cast<size_t>(cs.channels), 0.0f);
  if (mode == HC_RENDER_SPECTRAL) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) total += yb[i];
    for (int i = 0; i < n; ++i) cs.luma[static_cast<size_t>(i)] = static_cast<float>(yb[i] / total);
  } else if (mode == HC_RENDER_LATENT) {
    std::vector<double> col(static_cast<size_t>(k), 0.0);
    double total = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < k; ++j) col[static_cast<size_t>(j)] += yb[i] * c->Dd[static_cast<size_t>(i) * k + j];
    for (double v : col) total += v;
    if (total <= 0.0) total = 1.0;
    for (int j = 0; j < k; ++j) cs.luma[static_cast<size_t>(j)] = static_cast<float>(col[static_cast<size_t>(j)] / total);
  } else {
    cs.luma = {0.2126f, 0.7152f, 0.0722f};
  }
  // walls (renderer.cpp:149-159): left, right, floor, ceiling, back, front, inward normals
  const V3 a = v3(sc->box_min), b = v3(sc->box_max);
  const int* wm = sc->wall_material;
  cs.walls[0] = {0, a.x, a.y, b.y, a.z, b.z, {1, 0, 0}, wm[0]};
  cs.walls[1] = {0, b.x, a.y, b.y, a.z, b.z, {-1, 0, 0}, wm[1]};
  cs.walls[2] = {1, a.y, a.x, b.x, a.z, b.z, {0, 1, 0}, wm[2]};
  cs.walls[3] = {1, b.y, a.x, b.x, a.z, b.z, {0, -1, 0}, wm[3]};
  cs.walls[4] = {2, a.z, a.x, b.x, a.y, b.y, {0, 0, 1}, wm[4]};
  cs.walls[5] = {2, b.z, a.x, b.x, a.y, b.y, {0, 0, -1}, wm[5]};
  for (int i = 0; i < sc->n_objects; ++i) {
    const hc_scene_object& o = sc->objects[i];
    if (o.kind != 0 && o.kind != 1) fail("renderer: unknown object kind");
    cs.objects.push_back({o.kind, v3(o.center), o.radius, v3(o.box_min), v3(o.box_max), o.material});
  }
  return cs;
}

Frame camera_frame(const hc_scene* sc, int width, int height) {  // renderer.cpp:57-61
  Frame f;
  f.origin = v3(sc->cam_position);
  f.forward = normalize_h(sub(v3(sc->cam_look_at), f.origin));
  f.right = normalize_h(cross(f.forward, v3(sc->cam_up)));
  f.up = cross(f.right, f.forward);
  f.tan_half = std::tan(sc->cam_vfov_degrees * 3.14159265358979323846 / 360.0);
  f.aspect = static_cast<double>(width) / height;
  return f;
}

// slice_pass (renderer.cpp:274-283): one three-channel pass of a latent compile.
Compiled slice_pass(const Compiled& full, int pass) {
  Compiled cs = full;
  const int C = full.channels;
  cs.channels = 3;
  cs.eval_unit = 1;
  cs.luma = {1.0f / 3.0f, 1.0f / 3.0f, 1.0f / 3.0f};
  cs.albedo.clear();
  cs.emission.clear();
  for (size_t m = 0; m < full.albedo.size() / C; ++m)
    for (int q = 0; q < 3; ++q) cs.albedo.push_back(full.albedo[m * C + pass * 3 + q]);
  for (size_t l = 0; l < full.emission.size() / C; ++l)
    for (int q = 0; q < 3; ++q) cs.emission.push_back(full.emission[l * C + pass * 3 + q]);
  return cs;
}

template <class T>
struct DevVec {
  T* p = nullptr;
  ~DevVec() {
    if (p) cudaFree(p);
  }
  int put(const std::vector<T>& v, cudaStream_t s) {
    if (v.empty()) return HC_OK;
    HC_CUDA_TRY(cudaMalloc(&p, sizeof(T) * v.size()));
    HC_CUDA_TRY(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s));
    return HC_OK;
  }
};

// Pixel-serial launch when path hashes are collected, else sample-parallel in chunks of
// samples whose radiance buffers stay under ~256 MB.
template <int C>
int launch_render(hc_ctx ctx, const RenderParams& p) {
  const int64_t P = static_cast<int64_t>(p.width) * p.height;
  if (p.hashes) {
    render_kernel<C><<<static_cast<int>((P + 127) / 128), 128, 0, ctx->stream>>>(p);
    HC_CHECK_LAUNCH(ctx, "render_kernel");
    return HC_OK;
  }
  const int64_t per_sample = P * C * static_cast<int64_t>(sizeof(float));
  const int ns = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(p.spp, (int64_t(256) << 20) / per_sample)));
  int rc = ensure_scratch(ctx, static_cast<size_t>(P) * C * sizeof(double) + static_cast<size_t>(ns) * per_sample + 256);
  if (rc != HC_OK) return rc;
  double* accum = static_cast<double*>(ctx->scratch);
  float* samples = reinterpret_cast<float*>(static_cast<char*>(ctx->scratch) + ((P * C * sizeof(double) + 255) & ~size_t(255)));
  HC_CUDA_TRY(cudaMemsetAsync(accum, 0, sizeof(double) * P * C, ctx->stream));
  const int agrid = static_cast<int>(std::min<int64_t>((P * C + 255) / 256, int64_t(ctx->sm_count) * 16));
  for (int s0 = 0; s0 < p.spp; s0 += ns) {
    const int n = std::min(ns, p.spp - s0);
    render_samples_kernel<C><<<static_cast<int>((P * n + 127) / 128), 128, 0, ctx->stream>>>(p, s0, n, samples);
    HC_CHECK_LAUNCH(ctx, "render_samples_kernel");
    accumulate_kernel<C><<<agrid, 256, 0, ctx->stream>>>(samples, P, n, accum);
    HC_CHECK_LAUNCH(ctx, "accumulate_kernel");
  }
  finalize_kernel<<<agrid, 256, 0, ctx->stream>>>(accum, P * C, 1.0 / p.spp, p.image);
  HC_CHECK_LAUNCH(ctx, "finalize_kernel");
  return HC_OK;
}

// Render one compiled scene into image (H x W x cs.channels, device).
int render_compiled(hc_ctx ctx, const Compiled& cs, const hc_render_job* job, float* image, uint64_t* hashes,
                    unsigned long long* evals_dev) {
  DevVec<Object> dobj;
  DevVec<LightG> dl;
  DevVec<float> da, de, dluma;
  int rc;
  if ((rc = dobj.put(cs.objects, ctx->stream)) != HC_OK) return rc;
  if ((rc = dl.put(cs.lights, ctx->stream)) != HC_OK) return rc;
  if ((rc = da.put(cs.albedo, ctx->stream)) != HC_OK) return rc;
  if ((rc = de.put(cs.emission, ctx->stream)) != HC_OK) return rc;
  if ((rc = dluma.put(cs.luma, ctx->stream)) != HC_OK) return rc;
  RenderParams p;
  std::memset(&p, 0, sizeof(p));
  p.cam = cs.frame;
  for (int w = 0; w < 6; ++w) p.walls[w] = cs.walls[w];
  p.objects = dobj.p;
  p.n_objects = static_cast<int>(cs.objects.size());
  p.lights = dl.p;
  p.n_lights = static_cast<int>(cs.lights.size());
  p.albedo = da.p;
  p.emission = de.p;
  p.luma = dluma.p;
  p.width = job->width;
  p.height = job->height;
  p.spp = job->spp;
  p.max_depth = job->max_depth;
  p.seed = job->seed;
  p.eval_unit = cs.eval_unit;
  p.image = image;
  p.hashes = hashes;
  p.evals = evals_dev;
  switch (cs.channels) {
    case 3: rc = launch_render<3>(ctx, p); break;
    case 6: rc = launch_render<6>(ctx, p); break;
    case 9: rc = launch_render<9>(ctx, p); break;
    case 47: rc = launch_render<47>(ctx, p); break;
    case 81: rc = launch_render<81>(ctx, p); break;
    default: return set_error(HC_EUNSUPPORTED, "renderer: compiled for 3, 6, 9, 47 or 81 channels");
  }
  if (rc != HC_OK) return rc;
  HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));  // the scene tables are freed on return
  return HC_OK;
}

int check_job(const hc_render_job* job) {
  HC_REQUIRE(job, HC_EINVAL, "renderer: null job");
  HC_REQUIRE(job->width > 0 && job->height > 0 && job->spp > 0 && job->max_depth >= -1, HC_EINVAL,
             "renderer: invalid render job");
  return HC_OK;
}

__global__ void interleave_pass_kernel(const float* pass, int64_t P, int k, int b, float* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < P * 3; i += int64_t(gridDim.x) * blockDim.x)
    out[(i / 3) * k + 3 * b + i % 3] = pass[i];
}

}  // namespace
}  // namespace hcb

using namespace hcb;

extern "C" {

int hc_render(hc_codec codec, const hc_scene* scene, const hc_render_job* job, const double* d65, float* image,
              uint64_t* path_hashes, uint64_t* shading_evals) {
  HC_REQUIRE(codec && scene && image, HC_EINVAL, "renderer: null argument");
  int rc = check_job(job);
  if (rc != HC_OK) return rc;
  hc_ctx ctx = codec->ctx;
  try {
    Compiled cs = compile_scene(codec, scene, job->mode, d65);
    cs.frame = camera_frame(scene, job->width, job->height);
    DevVec<unsigned long long> evals;  // own buffer: render_compiled uses ctx->scratch
    if ((rc = evals.put(std::vector<unsigned long long>(1, 0ull), ctx->stream)) != HC_OK) return rc;
    rc = render_compiled(ctx, cs, job, image, path_hashes, evals.p);
    if (rc != HC_OK) return rc;
    if (shading_evals) HC_CUDA_TRY(cudaMemcpy(shading_evals, evals.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  } catch (const std::invalid_argument& e) {
    return set_error(HC_EINVAL, e.what());
  }
  return HC_OK;
}

int hc_render_latent_multipass(hc_codec codec, const hc_scene* scene, const hc_render_job* job, float* image,
                               uint64_t* path_hashes, uint64_t* shading_evals) {
  HC_REQUIRE(codec && scene && image, HC_EINVAL, "renderer: null argument");
  int rc = check_job(job);
  if (rc != HC_OK) return rc;
  hc_ctx ctx = codec->ctx;
  const int k = codec->k;
  const int64_t P = static_cast<int64_t>(job->width) * job->height;
  try {
    Compiled full = compile_scene(codec, scene, HC_RENDER_LATENT, nullptr);
    full.frame = camera_frame(scene, job->width, job->height);
    DevVec<unsigned long long> evals;  // own buffers: render_compiled uses ctx->scratch
    DevVec<float> pass_img;
    if ((rc = evals.put(std::vector<unsigned long long>(1, 0ull), ctx->stream)) != HC_OK) return rc;
    if ((rc = pass_img.put(std::vector<float>(static_cast<size_t>(3 * P), 0.0f), ctx->stream)) != HC_OK) return rc;
    for (int b = 0; b < k / 3; ++b) {  // renderer.cpp:641-657
      const Compiled pass = slice_pass(full, b);
      rc = render_compiled(ctx, pass, job, pass_img.p, b == 0 ? path_hashes : nullptr, evals.p);
      if (rc != HC_OK) return rc;
      interleave_pass_kernel<<<static_cast<int>(std::min<int64_t>((3 * P + 255) / 256, 4096)), 256, 0, ctx->stream>>>(
          pass_img.p, P, k, b, image);
      HC_CHECK_LAUNCH(ctx, "interleave_pass_kernel");
    }
    HC_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (shading_evals) HC_CUDA_TRY(cudaMemcpy(shading_evals, evals.p, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  } catch (const std::invalid_argument& e) {
    return set_error(HC_EINVAL, e.what());
  }
  return HC_OK;
}

}  // extern "C"
