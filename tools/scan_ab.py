"""Same-box A/B of the scan kernel between the current tree and another git
revision (default: round 1's 4a6aac6): builds tools/scan_ab/scan_ab.cu against
each tree's kernels.cu into its own .so, then alternates verify launches of
both on one random device buffer.  Run on the GPU box:

    python tools/scan_ab.py [REV] [MiB ...]
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build(tag, src_dir, extra):
    out = os.path.join(ROOT, "tools", "scan_ab", f"libscan_{tag}.so")
    cmd = ["nvcc", *ARCH, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-msse4.2", "-I", src_dir,
           "-I", os.path.join(ROOT, "include"), *extra, "-o", out,
           os.path.join(ROOT, "tools", "scan_ab", "scan_ab.cu"), os.path.join(src_dir, "crc_host.cpp")]
    subprocess.check_call(cmd)
    return out


def main():
    """`--build [REV]` (here, with git): build both libraries in tree (they
    travel to the GPU box with the snapshot); otherwise run them."""
    if len(sys.argv) > 1 and sys.argv[1] == "--build":
        rev = sys.argv[2] if len(sys.argv) > 2 else "4a6aac6"
        build("cur", os.path.join(ROOT, "paper_2502_16631_b200", "csrc"), [])
        old_dir = os.path.join(ROOT, "tools", "scan_ab", "old")
        os.makedirs(old_dir, exist_ok=True)
        for f in ("kernels.cu", "gcr_internal.h", "crc_host.cpp"):
            data = subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:paper_2502_16631_b200/csrc/{f}"])
            open(os.path.join(old_dir, f), "wb").write(data)
        has_basis = b"table_basis" in open(os.path.join(old_dir, "crc_host.cpp"), "rb").read()
        build("old", old_dir, [] if has_basis else ["-DSCAN_AB_R1"])
        full = subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short", rev]).decode().strip()
        open(os.path.join(ROOT, "tools", "scan_ab", "old", "REV"), "w").write(full)
        return
    rev = open(os.path.join(ROOT, "tools", "scan_ab", "old", "REV")).read().strip()
    sizes = [int(x) for x in sys.argv[1:]] or [1024, 4096]
    cur = os.path.join(ROOT, "tools", "scan_ab", "libscan_cur.so")
    old = os.path.join(ROOT, "tools", "scan_ab", "libscan_old.so")
    import torch
    libs = {"cur": C.CDLL(cur), "old": C.CDLL(old)}
    for L in libs.values():
        L.scan_ab_time.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_float)]
    for mib in sizes:
        n = mib << 20
        t = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        for P in (4096, 65536, 2097152):
            res = {"cur": [], "old": []}
            for rep in range(4):
                for k in ("old", "cur"):
                    ms = C.c_float()
                    assert libs[k].scan_ab_time(t.data_ptr(), n, P, 5, C.byref(ms)) == 0
                    res[k].append(round(ms.value * 1e3, 1))
            print({"MiB": mib, "P": P, "rev": rev, "us_old": res["old"], "us_cur": res["cur"],
                   "TBps_old": round(n / (min(res["old"]) * 1e-6) / 1e12, 3),
                   "TBps_cur": round(n / (min(res["cur"]) * 1e-6) / 1e12, 3)}, flush=True)
        del t


if __name__ == "__main__":
    main()
