"""Static SASS instruction mix of the hot kernels (cuobjdump -sass of the built library) ->
profiles/<tag>_sass_mix.txt.   python tools/sass_mix.py r02"""
import collections
import re
import subprocess
import sys

WANT = {"marg_stream_kernelILi0ELb1ELb0E": "marg_stream_kernel<0, Q32, no tail> (C4 a1)",
        "gather_dense_kernel": "gather_dense_kernel (a3)",
        "als_cluster_kernelILi10ELb1E": "als_cluster_kernel<10, GRID> (C4 a4)",
        "als_cluster_kernelILi10ELb0E": "als_cluster_kernel<10, cluster> (C2 a4)",
        "fitrows_kernelILi12E": "fitrows_kernel<12> (C4 a7)",
        "marg_coo_rep_kernelILi0ELb1E": "marg_coo_rep_kernel<0, VEC> (C5 a1)",
        "coo_gather_write_kernelILb1E": "coo_gather_write_kernel<SM> (C5 a3)",
        "coo_mttkrp_piece_kernelILi12E": "coo_mttkrp_piece_kernel<12> (C5 a4)"}


def main(tag):
    out = subprocess.run(["cuobjdump", "-sass", "paper_1709_00668_b200/libsambaten.so"],
                         capture_output=True, text=True).stdout
    want = dict(WANT)
    lines = ["# SASS instruction mix of the hot kernels (cuobjdump -sass of the built libsambaten.so; static",
             "# counts over the whole function, opcode without modifiers; tools/sass_mix.py).  Bulk copies and",
             "# mbarriers show as SYNCS / UBLKCP, warp sums as REDUX; no tensor-core (UTCMMA / HMMA) ops: the",
             "# path is integer, fp32 CUDA-core and HBM bound (DESIGN.md section 6).", ""]
    for f in re.split(r"\n\s+Function : ", out):
        name = f.split("\n", 1)[0].strip()
        for key, label in list(want.items()):
            if key in name:
                ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
                c = collections.Counter(o.split(".")[0] for o in ops)
                lines.append(f"## {label}: {sum(c.values())} instructions")
                lines.append("   " + ", ".join(f"{k} {v}" for k, v in c.most_common(24)))
                lines.append("")
                del want[key]
                break
    open(f"profiles/{tag}_sass_mix.txt", "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
