#!/usr/bin/env python
"""Instrument a copy of csrc/ds_merge.cu with per-warp / per-tile device printf traces of
the stage-3 kernels (union_links: units, shortcut / full-path units, words, links;
union_diag: fast path or tree merge) and build it into variants/trace.so.

    python tools/trace_patch.py && (on the GPU) cp variants/trace.so \
        paper_1506_02226_b200/libdensescan_b200.so && python tools/one_run.py
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_1506_02226_b200", "csrc")
TMP = "/tmp/ds_trace_src/paper_1506_02226_b200/csrc"
shutil.rmtree("/tmp/ds_trace_src", ignore_errors=True)
shutil.copytree(SRC, TMP)
os.makedirs("/tmp/ds_trace_src/include", exist_ok=True)
shutil.copy(os.path.join(ROOT, "include", "densescan_b200.h"), "/tmp/ds_trace_src/include/")
# every pipeline kernel: block 0 prints its name and start time right after griddep_wait
# (i.e. when its predecessor has completed); the label kernel's last block prints the end
h = os.path.join(TMP, "ds_internal.cuh")
hs = open(h).read()
anchor = """__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }"""
assert anchor in hs
hs = hs.replace(anchor, anchor + """
#define griddep_wait() do { asm volatile("griddepcontrol.wait;" ::: "memory"); \\
  if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_; \\
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); printf("KS %s %llu\\n", __func__, t_); } } while (0)""")
open(h, "w").write(hs)
STAMPS_ONLY = "--stamps-only" in sys.argv
p = os.path.join(TMP, "ds_merge.cu")
s = open(p).read()


ACTIVE = True


def rep(a, b, count=1):
    global s
    if not ACTIVE:
        return
    if a not in s:
        sys.exit(f"trace_patch: anchor not found: {a[:70]!r}")
    s = s.replace(a, b, count)


GT = 'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"'
rep("""        stamps[ST_LABELS_DONE] = t;""", """        stamps[ST_LABELS_DONE] = t;
        printf("KS end %llu\\n", t);""")
# union_links
ACTIVE = not STAMPS_ONLY  # the per-warp / per-tile traces below
rep("""  long long u = r_lo + (long long)blockIdx.x * LINK_WARPS + warp;
  int na = 0, nb = 0, nlb = 0;
  uint2 nce = make_uint2(0u, 0u);""", """  long long u = r_lo + (long long)blockIdx.x * LINK_WARPS + warp;
  unsigned long long t_start; """ + GT + """(t_start));
  int n_units = 0, n_uni = 0, n_full = 0, n_words = 0, n_links = 0, n_skipw = 0;
  int na = 0, nb = 0, nlb = 0;
  uint2 nce = make_uint2(0u, 0u);""")
rep("""    if (a == b) continue;  // round 1
    const uint32_t cnt""", """    if (a == b) continue;  // round 1
    ++n_units;
    const uint32_t cnt""")
rep("""        continue;
      }
    }
    // rows of the lane block""", """        ++n_uni;
        continue;
      }
    }
    ++n_full;
    // rows of the lane block""")
rep("""      if (skip_words) cc_any = wcnt > 0;""", """      if (skip_words) cc_any = wcnt > 0;
      n_words += wcnt; n_skipw += skip_words ? 1 : 0;""")
if ACTIVE:
    s = s.replace("link_root(parent, find_plain(parent, au), av);",
                  "link_root(parent, find_plain(parent, au), av); ++n_links;")
rep("""      __syncwarp();  // cols / groups / pair masks are rewritten by the next column block
    }
  }
}""", """      __syncwarp();  // cols / groups / pair masks are rewritten by the next column block
    }
  }
  for (int off = 16; off; off >>= 1) n_links += __shfl_xor_sync(0xffffffffu, n_links, off);
  unsigned long long t_end; """ + GT + """(t_end));
  if (lane == 0) printf("LT %d %d %llu %llu %d %d %d %d %d %d\\n", blockIdx.x, warp, t_start, t_end,
                        n_units, n_uni, n_full, n_words, n_links, n_skipw);
}""")
# union_diag: stamps after the setup, the word scatter and the column-minimum scan
rep("""  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int base = (int)tile * TILE;""", """  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    unsigned long long t_start, t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5 = 0, t4a = 0, t4b = 0, t4c = 0, t4d = 0; """ + GT + """(t_start));
#define DT(msg, ...) if (tid == 0) { unsigned long long t_end; """ + GT + """(t_end)); \\
    printf("DT %lld %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu " msg "\\n", (long long)tile, t_start, t1, t2, t3, t4, t5, t_end, t4a, t4b, t4c, t4d, __VA_ARGS__); }
    const int base = (int)tile * TILE;""")
rep("""    if (tid == 0) slot_root[0] = -1;  // atomicMax target of the single-root fast path
    __syncthreads();""", """    if (tid == 0) slot_root[0] = -1;  // atomicMax target of the single-root fast path
    __syncthreads();
    """ + GT + """(t1));""")
rep("""    __syncthreads();
    // minimum neighbour of every core column""", """    __syncthreads();
    """ + GT + """(t2));
    // minimum neighbour of every core column""")
rep("""        lp[ww * 32 + l] = q0 * RB + r;
      }
    }
    __syncthreads();""", """        lp[ww * 32 + l] = q0 * RB + r;
      }
    }
    __syncthreads();
    """ + GT + """(t3));""")
rep("""        __syncthreads();  // smem is reused by the next tile
        continue;""", """        DT("fast %d 0", nentries)
        __syncthreads();  // smem is reused by the next tile
        continue;""")
rep("""      const int64_t g = (int64_t)base + v;
      int r = -1;
      if (g < n) {
        r = find_local(lp, v);""", """      const int64_t g = (int64_t)base + v;
      DT("slow %d %d", nentries, ntrees)
      int r = -1;
      if (g < n) {
        r = find_local(lp, v);""")
rep("""      if (!__syncthreads_or(nv != cur)) break;
    }""", """      if (!__syncthreads_or(nv != cur)) break;
    }
    """ + GT + """(t4));""")
rep("""    __syncthreads();
    {
      const int v = tid;""", """    __syncthreads();
    """ + GT + """(t5));
    {
      const int v = tid;""")

# tree-merge sub-phases (slow tiles): slots assigned, tree masks, crossing scan, closure
rep("""      if (k < 32) slot_root[k] = tid;    // slot -> root node
    }
    __syncthreads();""", """      if (k < 32) slot_root[k] = tid;    // slot -> root node
    }
    __syncthreads();
    """ + GT + """(t4a));""")
rep("""        if (is_core && (tid & 31) == __ffs(grp) - 1) M[key * WPR + (tid >> 5)] = __brev(grp);
      }
      __syncthreads();""", """        if (is_core && (tid & 31) == __ffs(grp) - 1) M[key * WPR + (tid >> 5)] = __brev(grp);
      }
      __syncthreads();
      """ + GT + """(t4b));""")
rep("""        atomicOr(&adj[k], bits);
      }
      __syncthreads();""", """        atomicOr(&adj[k], bits);
      }
      __syncthreads();
      """ + GT + """(t4c));""")
rep("""        adj[tid] = row;
      }
      __syncthreads();""", """        adj[tid] = row;
      }
      __syncthreads();
      """ + GT + """(t4d));""")
open(p, "w").write(s)
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
r = subprocess.run(["make", "-s", "-C", TMP, "OUT=" + os.path.join(ROOT, "variants", "trace.so"),
                    "OBJDIR=/tmp/ds_trace_obj"], capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print("built variants/trace.so")
