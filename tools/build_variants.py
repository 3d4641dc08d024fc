"""Build tuning variants of libkmeans.so into tune/ (KMEANS_LIB_OVERRIDE selects one)."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
from paper_2405_12052_b200 import build as kb

VARIANTS = {
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
    "rg128": ("KM_ROW_GROUP=128",),
    "rg256": ("KM_ROW_GROUP=256",),
    "rg512": ("KM_ROW_GROUP=512",),
    "rg1024": ("KM_ROW_GROUP=1024",),
    "nowrite": ("KM_EXP_NOWRITE=1",),   # timing experiment only (wrong results)
    "sg128": ("KM_SPARSE_GROUP=128",),
    "sg256": ("KM_SPARSE_GROUP=256",),
    "m32": ("KM_MORTON32=1",),
    "m64": ("KM_MORTON32=0",),
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
    "ls4": ("KM_LARGE_SLOTS=4",),
    "ls16": ("KM_LARGE_SLOTS=16",),
    "lc32": ("KM_LARGE_CAP=32",),
    "lc128": ("KM_LARGE_CAP=128",),
    "pdl0": ("KM_PDL=0",),
    "pdl1": ("KM_PDL=1",),
    "pdl1t": ("KM_PDL=1", "KM_PDL_ASSIGN_TRIGGER=1"),
}
if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        print(kb.build(force=True, out=f"tune/libkmeans_{n}.so", defines=VARIANTS[n]))
