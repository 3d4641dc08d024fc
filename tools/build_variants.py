"""Build tuning variants of libkmeans.so into tune/ (KMEANS_LIB_OVERRIDE selects one)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2405_12052_b200 import build as kb

VARIANTS = {
    "lnpl1": ("KM_LARGE_NPL2=0",),    # k_assign_large: 4 points per lane at every K
    "lk16": ("KM_LARGE_KT=16",),      # k_assign_large: 16 centroids per argmin step
    "lnpl3": ("KM_LARGE_NPL_BIG=3",),  # k_assign_large: 12 points per lane at large K
    "lu2": ("KM_LARGE_UNROLL=2",),     # k_assign_large: two argmin steps per loop trip
    "aggbfly": ("KM_AGG_TRANSPOSE=0",),      # pruned slot sums: plain 5-level butterflies
    "aggtile": ("KM_AGG_UNIT=0",),             # pruned, large K: slot sums per warp-tile
    "hprof": ("KM_HEAVY_PROF=1",),
    "ru1": ("KM_REFINE_UNROLL=1",),            # list refinement loops not unrolled             # per-chunk phase times of k_assign_heavy (printf)
    "sup16": ("KM_SUPER_CHUNKS=16",),          # large K: 16 chunks per prune super box
    "sup32": ("KM_SUPER_CHUNKS=32",),
    "sup128": ("KM_SUPER_CHUNKS=128",),
    "lfwd": ("KM_LARGE_REVERSE=0",),          # large-K pruned kernel: chunks in curve order
    "htold": ("KM_HEAVY_TILES=0",),            # heavy chunks: one block per chunk (k_assign_heavy)
    "hnog": ("KM_HEAVY_GATHER=0",),            # heavy tiles: walk through the tile list (no gathered centroids)
    "htb3": ("KM_HEAVY_TILE_MINB=3",),         # k_assign_heavy_tiles: <= 85 registers
    "htb4": ("KM_HEAVY_TILE_MINB=4",),         # k_assign_heavy_tiles: <= 64 registers
    "lnosplit": ("KM_LARGE_SPLIT_WARPS=0",),   # large K: never split into labels + accumulate
    "lsnpl1": ("KM_LARGE_SPLIT_NPL=1",),       # split labels pass: 4 points per lane
    "lsnpl2": ("KM_LARGE_SPLIT_NPL=2",),       # split labels pass: 8 points per lane
    "lnb3": ("KM_LARGE_NPL_BIG=3",),           # fused, one block per SM: 12 points per lane
    "lsplit64": ("KM_LARGE_SPLIT_WARPS=64",),  # split at every large K
    "lsplit12": ("KM_LARGE_SPLIT_WARPS=12",),  # split below 12 fused warps per SM
    "base": (),
    "c32": ("KM_CHUNK_TILES=32",),
    "st6": ("KM_SORTED_STAGES=6",),
    "st3": ("KM_SORTED_STAGES=3",),
    "c32st6": ("KM_CHUNK_TILES=32", "KM_SORTED_STAGES=6"),
    "sl2": ("KM_SORTED_SLOTS=2",),
    "c8": ("KM_CHUNK_TILES=8",),
    "u1st3": ("KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=3"),
    "u1st4": ("KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=4"),
    "u1st6": ("KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=6"),
    "c8st3": ("KM_CHUNK_TILES=8", "KM_SORTED_STAGES=3"),
    "c8u1st4": ("KM_CHUNK_TILES=8", "KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=4"),
    "st2": ("KM_SORTED_STAGES=2",),
    "c4u1st4": ("KM_CHUNK_TILES=4", "KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=4"),
    "c4st2": ("KM_CHUNK_TILES=4", "KM_SORTED_STAGES=2"),
    "c8u1st3": ("KM_CHUNK_TILES=8", "KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=3"),
    "c8st2": ("KM_CHUNK_TILES=8", "KM_SORTED_STAGES=2"),
    "c2u1st2": ("KM_CHUNK_TILES=2", "KM_SORTED_UNIT_SUB=1", "KM_SORTED_STAGES=2"),
    "rg64": ("KM_ROW_GROUP=64",),
    "rg128": ("KM_ROW_GROUP=128",),
    "rg256": ("KM_ROW_GROUP=256",),
    "rg512": ("KM_ROW_GROUP=512",),
    "rg1024": ("KM_ROW_GROUP=1024",),
    "sg32": ("KM_SPARSE_GROUP=32",),
    "sg64": ("KM_SPARSE_GROUP=64",),
    "sg128": ("KM_SPARSE_GROUP=128",),
    "sg256": ("KM_SPARSE_GROUP=256",),
    "m32": ("KM_MORTON32=1",),
    "zcurve": ("KM_HILBERT=0",),
    "nobis": ("KM_BISECTOR=0",),   # box test only (round 1's pruning)
    "m64": ("KM_MORTON32=0",),
    "sct4": ("KM_SORTED_CHUNK_TILES=4",),
    "sct4rg512": ("KM_SORTED_CHUNK_TILES=4", "KM_ROW_GROUP=512"),
    "sct8": ("KM_SORTED_CHUNK_TILES=8",),
    "bc16": ("KM_BIG_CHUNK_TILES=16",),
    "bc32": ("KM_BIG_CHUNK_TILES=32",),
    "mx4": ("KM_MORTON_EXTRA=4",),
    "mx6": ("KM_MORTON_EXTRA=6",),
    "tpw1": ("KM_FUSED_TPW=1",),
    "tpw2": ("KM_FUSED_TPW=2",),
    "tpw4": ("KM_FUSED_TPW=4",),
    "tpw8": ("KM_FUSED_TPW=8",),
    "tpw16": ("KM_FUSED_TPW=16",),
    "tpw32": ("KM_FUSED_TPW=32",),
    "cu0": ("KM_CAND_UNROLL2=0",),
    "cu1": ("KM_CAND_UNROLL2=1",),
    "ef0": ("KM_EVICT_FIRST=0",),
    "ef1": ("KM_EVICT_FIRST=1",),
    "cm10": ("KM_CHUNK_MINB=10",),
    "cm12": ("KM_CHUNK_MINB=12",),
    "cm16": ("KM_CHUNK_MINB=16",),
    "mb1": ("KM_PRUNED_MINB=1",),
    "mb20": ("KM_PRUNED_MINB=20",),
    "mb26": ("KM_PRUNED_MINB=26",),
    "mb24": ("KM_PRUNED_MINB=24",),
    "mb28": ("KM_PRUNED_MINB=28",),
    "mb32": ("KM_PRUNED_MINB=32",),
    "tc0": ("KM_TWO_CAND=0",),
    "tc1": ("KM_TWO_CAND=1",),
    "pdl0": ("KM_PDL=0",),
    "pdl1": ("KM_PDL=1",),
    "pdl1t": ("KM_PDL=1", "KM_PDL_ASSIGN_TRIGGER=1"),
    "pdlt": ("KM_PDL_ASSIGN_TRIGGER=1",),
    "checked": ("KM_CHECKS=1",),
    "lmb16": ("KM_PRUNED_MINB_LARGE=16",),
    "tcp0": ("KM_TWO_CAND_PRED=0",),
    "lmb24": ("KM_PRUNED_MINB_LARGE=24",),
    "lc32": ("KM_LARGE_CAP=32",),
    "pw24": ("KM_PERSIST_WARPS_3D=24", "KM_PERSIST_WARPS_2D=24"),
    "pw20": ("KM_PERSIST_WARPS_3D=20", "KM_PERSIST_WARPS_2D=20"),
    "pnw": ("KM_PERSIST_NOWAIT=1",),   # timing experiment: the persistent kernel without its flag waits
    "pnw20": ("KM_PERSIST_NOWAIT=1", "KM_PERSIST_WARPS_3D=20", "KM_PERSIST_WARPS_2D=20"),   # device bounds checks + red zones (stand-in for compute-sanitizer)
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        print(kb.build(force=True, out=f"tune/libkmeans_{n}.so", defines=VARIANTS[n]))
