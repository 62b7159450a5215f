"""Resource budgets of the default hot-path kernels, read from the ptxas
report the build writes (paper_1708_01873_b200/csrc/ptxas.log).

Occupancy is a measured choice for every default kernel
and it can silently shift with unrelated source changes: an explicit
__launch_bounds__ minimum of 1 once let ptxas give the float64 rectangular
tiles 168 registers instead of 122 -- 1 CTA/SM instead of 2, -15 % at cfg3-8
(profiles/r02_rect_minb_ab.jsonl).  These checks need no GPU; without a
build report they skip."""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

LOG = Path(__file__).resolve().parents[1] / "paper_1708_01873_b200" / "csrc" / "ptxas.log"

# demangled-name prefix -> (max registers, CTAs/SM the default relies on)
BUDGETS = {
    "bitrev_oop_tile_kernel<16, 6, 256, true, 1>": (255, 1),      # cfg3-16
    "bitrev_oop_rect_kernel<8, 7, 5, true>": (128, 2),            # cfg3-8, cfg5
    "bitrev_oop_rect_kernel<8, 8, 5, false>": (255, 1),           # cfg4 (batched rows tier)
    "bitrev_oop_rect_kernel<4, 8, 6, true>": (255, 1),            # cfg3-4
    "bitrev_inplace_tile_kernel<8, 6, true, true>": (255, 1),     # cfg2
    "bitrev_ring_kernel<16, 4, false, 2, false>": (128, 2),       # cfg1 (TMA tensor ring)
    "bitrev_fft_rect_kernel<8, 7, 5, 7>": (128, 2),               # cfg4-fft7
    "bitrev_pack_rect_kernel<8, 7, 5>": (128, 2),                 # cfg5 pack
    "sharded_unpack_kernel<8, 8>": (128, 2),                      # cfg5 unpack
}


def _entries():
    if not LOG.exists():
        pytest.skip("no ptxas report: build the library first")
    text = LOG.read_text()
    ents = re.findall(r"Compiling entry function '(\S+)' for 'sm_100a'\n"
                      r"ptxas info\s+: Function properties for \S+\n"
                      r"\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n"
                      r"ptxas info\s+: Used (\d+) registers", text)
    if not ents:
        pytest.skip("ptxas report has no entries")
    filt = shutil.which("c++filt")
    if not filt:
        pytest.skip("c++filt not available")
    names = subprocess.run([filt], input="\n".join(e[0] for e in ents), capture_output=True,
                           text=True, check=True).stdout.splitlines()
    out = {}
    for (_, stack, spill_st, spill_ld, regs), dem in zip(ents, names):
        key = dem.split("bitrev_b200::", 1)[-1]
        out[key] = (int(regs), int(spill_st) + int(spill_ld), int(stack))
    return out


@pytest.mark.parametrize("prefix", sorted(BUDGETS))
def test_default_kernel_budget(prefix):
    ents = _entries()
    hits = [v for k, v in ents.items() if k.startswith(prefix)]
    assert hits, f"{prefix} not in the ptxas report"
    max_regs, ctas = BUDGETS[prefix]
    for regs, spills, _ in hits:
        assert spills == 0, f"{prefix}: {spills} bytes of spills"
        assert regs <= max_regs, f"{prefix}: {regs} registers > {max_regs} ({ctas} CTAs/SM)"
        assert regs * 256 * ctas <= 65536, f"{prefix}: {regs} registers do not fit {ctas} CTAs/SM"


# single-CTA in-place pairs of 1 KB-row tiles: kept as tuning paths only
# (they spill at 255 registers, which is why complex128 in
# place defaults to the 2-CTA cluster pairs and float32 in place to Q6)
TUNING_ONLY = ("bitrev_inplace_tile_kernel<16, 6,", "bitrev_inplace_tile_kernel<4, 7,")


def test_no_spills_in_default_tile_kernels():
    """No instantiation of the permutation tile kernels spills, except the
    documented tuning-only in-place shapes."""
    ents = _entries()
    fams = ("bitrev_oop_tile_kernel", "bitrev_oop_rect_kernel", "bitrev_inplace_tile_kernel",
            "bitrev_rows_kernel", "bitrev_pack_rect_kernel")
    bad = {k: v for k, v in ents.items()
           if k.startswith(fams) and not k.startswith(TUNING_ONLY) and v[1]}
    assert not bad, bad
