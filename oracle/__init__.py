"""CPU oracle (test infrastructure only; see ref_cpu_exec.h)."""
