"""INTEGRATION.md §1 is real code: its C++ adapter is compiled against the reference's own
headers (this container only) and driven with a reference-built GridSchedule through the C-ABI.
The schedule must round-trip unchanged (pb_schedule_create validates like validate_schedule),
and without a GPU the executor call must fail loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/include"
JSON = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"

MAIN = r'''
#include <cstdio>
#include <cstring>
int main() {
    auto g = pipeblock::assemble(pipeblock::build_entry("v-half", 4), 8);
    std::vector<pb_pass> passes;
    for (const auto& p : g.passes)
        passes.push_back({p.device, p.stage, int32_t(p.kind), p.microbatch, p.start, p.duration});
    pb_topology topo{g.topology.devices, g.topology.num_stages, g.topology.placement.data(),
                     g.topology.stage_mem.data()};
    pb_schedule* s = nullptr;
    if (pb_schedule_create(&topo, passes.data(), passes.size(), g.microbatches, &s) != PB_OK) return 2;
    std::vector<pb_pass> back(passes.size());
    if (pb_schedule_passes(s, back.data(), back.size()) != PB_OK) return 3;
    for (size_t i = 0; i < back.size(); ++i)
        if (std::memcmp(&back[i], &passes[i], sizeof(pb_pass)) != 0) return 4;
    double peaks[4];
    pb_schedule_exact_peak(s, peaks);
    auto ref = pipeblock::exact_peak(g);
    for (int d = 0; d < 4; ++d)
        if (peaks[d] != ref.per_device[d]) return 5;
    pb_model_cfg cfg{2, 256, 2, 256, 512, 1, 1, 1e-3f, 0.9f, 0.95f, 1e-8f, 0.f, 1, 0, nullptr};
    std::vector<int32_t> tok(8 * 256, 1), lab(8 * 256, 2);
    try {
        execute_on_b200(g, cfg, 1, 0, tok.data(), lab.data());
        return 6;  // no GPU here: must not succeed
    } catch (const std::runtime_error& e) {
        std::printf("executor refused: %s\n", e.what());
    }
    pb_schedule_destroy(s);
    std::printf("INTEGRATION_OK %zu passes\n", passes.size());
    return 0;
}
'''


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference headers not mounted")
def test_integration_adapter_compiles_and_round_trips(tmp_path):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```cpp\n(.*?)```", text, re.S).group(1)
    src = tmp_path / "adapter.cpp"
    src.write_text("#include <stdexcept>\n#include <vector>\n" + block + MAIN)
    exe = tmp_path / "adapter"
    lib_dir = os.path.join(ROOT, "paper_2405_15362_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF}", f"-I{JSON}", f"-I{ROOT}/include", str(src), "-o", str(exe),
                    f"-L{lib_dir}", "-l:libpb200.so", f"-Wl,-rpath,{lib_dir}"], check=True, capture_output=True,
                   text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "INTEGRATION_OK" in r.stdout
