#!/usr/bin/env python
"""Kernel timeline build: every block of every pipeline kernel records (file, line of its
griddep_wait, block) and %globaltimer right after griddep_wait into mapped page-locked
memory; ds_run_dbscan appends each call's records to $DS_KT_OUT. Builds variants/kt.so
from a patched copy of csrc/ (the product sources are not touched).

    python tools/kt_patch.py
    (GPU) cp variants/kt.so paper_1506_02226_b200/libdensescan_b200.so
          DS_KT_OUT=gpurun_out/kt.txt DS_RUNS=4 python tools/one_run.py
    python tools/kt_report.py gpurun_out/kt.txt
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1506_02226_b200", "csrc")
BASE = "/tmp/ds_kt_src"
TMP = BASE + "/paper_1506_02226_b200/csrc"
shutil.rmtree(BASE, ignore_errors=True)
shutil.copytree(SRC, TMP)
os.makedirs(BASE + "/include", exist_ok=True)
shutil.copy(os.path.join(ROOT, "include", "densescan_b200.h"), BASE + "/include/")

FILES = ["ds_tile.cu", "ds_merge.cu", "ds_sort.cu", "ds_dist.cu", "ds_closure.cu", "ds_serial.cu",
         "ds_api.cu"]
KT_CAP = 1 << 20  # u64 words

h = os.path.join(TMP, "ds_internal.cuh")
hs = open(h).read()
anchor = """__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }"""
assert anchor in hs
hs = hs.replace(anchor, anchor + f"""
namespace kt {{
__device__ unsigned long long* g_kt;  // per translation unit, set by ds_kt_set_<file>
}}
#define griddep_wait() do {{ asm volatile("griddepcontrol.wait;" ::: "memory"); \\
  if (threadIdx.x == 0 && ::ds::kt::g_kt) {{ unsigned long long t_; \\
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \\
    const unsigned i_ = atomicAdd(reinterpret_cast<unsigned*>(::ds::kt::g_kt), 2u); \\
    if (i_ + 4 < {KT_CAP}u) {{ \\
      ::ds::kt::g_kt[2 + i_] = ((unsigned long long)KT_FILE << 48) | ((unsigned long long)__LINE__ << 32) | blockIdx.x; \\
      ::ds::kt::g_kt[3 + i_] = t_; }} }} }} while (0)""")
hs = hs.replace("#define griddep_wait()", """#define KT_MARK(site) do { if (::ds::kt::g_kt) { unsigned long long t_; \\
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); \\
    const unsigned i_ = atomicAdd(reinterpret_cast<unsigned*>(::ds::kt::g_kt), 2u); \\
    if (i_ + 4 < """ + str(KT_CAP) + """u) { \\
      ::ds::kt::g_kt[2 + i_] = ((unsigned long long)KT_FILE << 48) | ((unsigned long long)(site) << 32) | \\
                               (blockIdx.x * 32u + (threadIdx.x >> 5)); \\
      ::ds::kt::g_kt[3 + i_] = t_; } } } while (0)
#define griddep_wait()""", 1)
open(h, "w").write(hs)

# DS_KT_PHASES=1: thread 0 of every union_diag CTA also stamps its phase boundaries
# (sites 61001..), reported by tools/kt_phases.py
PHASES = [
    (61001, "    if (tid == 0) slot_root[0] = -1;  // atomicMax target of the single-root fast path\n    __syncthreads();", True),
    (61002, "    // minimum neighbour of every core column", False),
    (61003, "    // Fast path: a core point without a smaller core neighbour", False),
    (61004, "        __syncthreads();  // smem is reused by the next tile\n        continue;", False),
    (61005, "    // merge the min-neighbour trees.", False),
    (61006, "    __syncthreads();\n    {\n      const int v = tid;", True),
    (61007, "    __syncthreads();\n  }\n}\n\n// Round 2, off-diagonal", False),
    (61008, "      for (int r = 0; r < RB; ++r) {\n        const int u = cblk * RB + r;\n        uint32_t um = R[w * DIAG_RS + u];", False),
    (61009, "      auto locate = [&](int j) -> unsigned long long {", False),
    (61010, "      for (int r = 0; r < RB; ++r) {\n        const int u = cblk * RB + r;\n        const uint32_t um = R[w * DIAG_RS + u];", False),
    (61011, "      if (tid < 32) {  // symmetric transitive closure", False),
    # union_links: per-warp end (61100)
    (61101, "    const int a = na, b = nb, lb = nlb;\n    const uint2 ce = nce;", False),
    (61100, "      __syncwarp();  // cols / groups / pair masks are rewritten by the next column block\n    }\n  }", True),
]
for fi, f in enumerate(FILES):
    p = os.path.join(TMP, f)
    s = open(p).read()
    name = f[3:-3]
    s = f"#define KT_FILE {fi}\n" + s + f"""
extern "C" void ds_kt_set_{name}(void* p) {{ cudaMemcpyToSymbol(ds::kt::g_kt, &p, sizeof p); }}
"""
    if f == "ds_tile.cu":  # per-warp end of the eps kernel: site 60000
        anchor = """  flush();
  if (lane == 0 && steps_done)"""
        assert anchor in s
        s = s.replace(anchor, """  flush();
  if (lane == 0) KT_MARK(60000);
  if (lane == 0 && steps_done)""", 1)
    if f == "ds_merge.cu" and os.environ.get("DS_KT_PHASES"):  # union_diag phase marks
        M = lambda site: (f"if (threadIdx.x == 0) KT_MARK({site});" if site < 61100 else
                          f"if ((threadIdx.x & 31) == 0) KT_MARK({site});")
        for site, anchor, after in PHASES:
            if anchor not in s:
                print("kt_patch: phase anchor not found, site", site, "skipped")
                continue
            s = s.replace(anchor, anchor + "\n" + M(site) if after else M(site) + "\n" + anchor, 1)
    if f == "ds_api.cu":
        decl = "".join(f'extern "C" void ds_kt_set_{g[3:-3]}(void* p);\n' for g in FILES)
        s = s.replace('#include "ds_internal.cuh"', '#include "ds_internal.cuh"\n#include <cstdio>\n#include <cstdlib>\n' + decl, 1)
        old = """  st = pipeline(c, (const double*)c->coords64.p, n, d, eps_sq, min_pts, formula, mem_cap,
                (int64_t*)c->labels.p, counts_out ? (int64_t*)c->counts64.p : nullptr, s, &local,
                &io);"""
        assert old in s
        setall = "".join(f"ds_kt_set_{g[3:-3]}(dp); " for g in FILES)
        new = f"""  static unsigned long long* kt_d = nullptr;
  static unsigned long long* kt_h = nullptr;
  if (!kt_d && getenv("DS_KT_OUT")) {{
    cudaMalloc((void**)&kt_d, {KT_CAP} * 8);
    kt_h = (unsigned long long*)malloc({KT_CAP} * 8);
    void* dp = kt_d;
    {setall}
  }}
  if (kt_d) cudaMemsetAsync(kt_d, 0, 8, c->stream);
""" + old + f"""
  if (kt_d) {{
    cudaDeviceSynchronize();
    cudaMemcpy(kt_h, kt_d, {KT_CAP} * 8, cudaMemcpyDeviceToHost);
    FILE* fo = fopen(getenv("DS_KT_OUT"), "a");
    const unsigned m = (unsigned)kt_h[0] < {KT_CAP} - 4 ? (unsigned)kt_h[0] : {KT_CAP} - 4;
    fprintf(fo, "CALL %lld\\n", (long long)n);
    for (unsigned i = 0; i < m; i += 2)
      fprintf(fo, "%llu %llu %llu %llu\\n", kt_h[2 + i] >> 48, (kt_h[2 + i] >> 32) & 0xffff,
              kt_h[2 + i] & 0xffffffffu, kt_h[3 + i]);
    fclose(fo);
  }}"""
        s = s.replace(old, new, 1)
    open(p, "w").write(s)

os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
r = subprocess.run(["make", "-s", "-C", TMP, "OUT=" + os.path.join(ROOT, "variants", "kt.so"),
                    "OBJDIR=/tmp/ds_kt_obj"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout[-3000:] + r.stderr[-3000:])
# kernel names by (file, line): the kernel enclosing each griddep_wait call
names = {}
import re
for fi, f in enumerate(FILES):  # line numbers of the patched copy (what __LINE__ saw)
    lines = open(os.path.join(TMP, f)).read().split("\n")
    cur = None
    for ln, l in enumerate(lines, start=1):
        m = re.search(r"__global__ void(?: __launch_bounds__\([^)]*\))? (\w+)", l)
        if m:
            cur = m.group(1)
        if "griddep_wait();" in l and cur:
            names[f"{fi}:{ln}"] = cur
names["0:60000"] = "eps_warp_end"
with open(os.path.join(ROOT, "variants", "kt_names.txt"), "w") as fo:
    for k, v in names.items():
        fo.write(f"{k} {v}\n")
print("built variants/kt.so;", len(names), "kernel sites")
