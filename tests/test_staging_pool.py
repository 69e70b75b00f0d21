"""csrc/staging.h's WorkerPool (the host worker threads of the staged
geometry upload): every item runs exactly once per run(), back-to-back runs
with different sizes and bodies, zero-item runs, and runs after the workers
went idle -- compiled and run on the CPU (the CUDA headers are present here;
nothing CUDA is called)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SRC = r"""
#include "staging.h"
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
int main() {
  pgpu::WorkerPool pool(7);
  long long expect = 0, got = 0;
  for (int rep = 0; rep < 2000; ++rep) {
    const int n = rep % 37;  // includes 0
    std::vector<std::atomic<int>> hits(n > 0 ? n : 1);
    for (auto& h : hits) h.store(0);
    std::atomic<long long> sum{0};
    pool.run(n, [&](int i) { hits[i].fetch_add(1); sum.fetch_add(i + rep); });
    for (int i = 0; i < n; ++i)
      if (hits[i].load() != 1) { std::printf("item %d ran %d times\n", i, hits[i].load()); return 1; }
    for (int i = 0; i < n; ++i) expect += i + rep;
    got += sum.load();
    if (rep % 500 == 0) std::this_thread::sleep_for(std::chrono::milliseconds(5));  // idle workers
  }
  if (expect != got) { std::printf("sum mismatch\n"); return 2; }
  std::printf("ok\n");
  return 0;
}
"""


def test_worker_pool(tmp_path):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no g++")
    src = tmp_path / "pool_test.cpp"
    src.write_text(SRC)
    exe = tmp_path / "pool_test"
    build = subprocess.run([cxx, "-std=c++17", "-O2", "-pthread",
                            f"-I{ROOT / 'paper_1507_06565_b200' / 'csrc'}", "-I/usr/local/cuda/include",
                            str(src), "-o", str(exe)], capture_output=True, text=True)
    assert build.returncode == 0, build.stderr[-2000:]
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0 and res.stdout.strip() == "ok", res.stdout + res.stderr
