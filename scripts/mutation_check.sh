#!/bin/bash
# Mutation check of the GPU parity suite (run on a GPU box from the repo root): build copies of
# libeva.so with one deliberate bug each and require that the named tests FAIL against them
# (EVA_LIB_PATH loads the mutant).  Prints one line per mutant: KILLED (tests failed, good) or
# SURVIVED (the suite cannot see the bug).
set -u
ROOT=$(pwd)
run_mutant() {  # name file sed-expr pytest-selection
  local name=$1 file=$2 expr=$3 sel=$4
  local dir=/tmp/mut_$name
  rm -rf "$dir"; mkdir -p "$dir"
  cp -r "$ROOT/paper_2511_00576_b200" "$ROOT/include" "$dir/"
  rm -rf "$dir/paper_2511_00576_b200/build" "$dir/paper_2511_00576_b200/libeva.so"
  sed -i "$expr" "$dir/paper_2511_00576_b200/csrc/$file"
  if cmp -s "$ROOT/paper_2511_00576_b200/csrc/$file" "$dir/paper_2511_00576_b200/csrc/$file"; then
    echo "MUTANT $name: sed did not apply"; return
  fi
  (cd "$dir" && python -c "import sys; sys.path.insert(0,'paper_2511_00576_b200'); import build; build.build()") \
    > "$dir/build.log" 2>&1 || { echo "MUTANT $name: build failed"; tail -5 "$dir/build.log"; return; }
  EVA_LIB_PATH="$dir/paper_2511_00576_b200/libeva.so" ${MUT_ENV:-} timeout 900 \
    python -m pytest tests -q -m gpu -x -k "$sel" -p no:cacheprovider > "$dir/test.log" 2>&1
  local rc=$?
  if [ $rc -eq 0 ]; then echo "MUTANT $name: SURVIVED ($(tail -1 "$dir/test.log"))";
  else echo "MUTANT $name: KILLED ($(grep -m1 -E '^FAILED|Error' "$dir/test.log" | cut -c1-160))"; fi
}
# Eq.15 gate of the register finalize (unfused schedule and the fused schedule's COEF mode)
run_mutant gate_deleted backward_simt.cu \
  's/sh_g\[j\] = (x >= -cfg.clip \&\& x <= cfg.clip) ? cfg.lambda : 0.f;/sh_g[j] = cfg.lambda;/' \
  "test_backward_bf16_omega_branch"
run_mutant gate_lambda_one backward_simt.cu \
  's/sh_g\[j\] = (x >= -cfg.clip \&\& x <= cfg.clip) ? cfg.lambda : 0.f;/sh_g[j] = (x >= -cfg.clip \&\& x <= cfg.clip) ? 1.0f : 0.f;/' \
  "test_backward_bf16_omega_branch"
MUT_ENV="env EVA_BACKWARD_FUSED=1" run_mutant gate_deleted_fused backward_simt.cu \
  's/sh_g\[j\] = (x >= -cfg.clip \&\& x <= cfg.clip) ? cfg.lambda : 0.f;/sh_g[j] = cfg.lambda;/' \
  "test_backward_bf16_omega_branch"
# split-K merge counter placed after the partials again
run_mutant counters_after_partials kernels_simt.cu \
  's|unsigned\* counters = reinterpret_cast<unsigned\*>(ws);|unsigned* counters = reinterpret_cast<unsigned*>(ws + ((size_t)gridDim.x + 3) / 4 * 4 + (size_t)gridDim.x * S * (D + 2));|' \
  "test_decode_split_count_changes"
