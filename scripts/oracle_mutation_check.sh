#!/usr/bin/env bash
# Mutation check for the oracle's pins: each mutation is a plausible mistake in
# oracle/cce_oracle.c; the pin suite must fail for every one of them.
set -u
cd "$(dirname "$0")/.."
cp oracle/cce_oracle.c /tmp/oracle_orig.c
trap 'cp /tmp/oracle_orig.c oracle/cce_oracle.c; python -c "import oracle; oracle.build(force=True)"' EXIT
muts=(
 's/(v == y ? 1.0 : 0.0)/(v == y ? 0.0 : 0.0)/'                       # dropped one-hot
 's/dloss \/ (double)nv/dloss \/ (double)N/'                           # wrong mean divisor
 's/for (int64_t v = 0; v < V; ++v) s += exp(z\[v\] - m);/for (int64_t v = 1; v < V; ++v) s += exp(z[v] - m);/'  # dropped term
 's/out\[d\] += g \* hr\[d\];/out[d] += g * w[d];/'                   # transposed operand in dW
 's/row_loss\[n\] = l - z\[y\];/row_loss[n] = l + z[y];/'             # sign
 's/return m + log(s);/return log(s);/'                                # dropped max shift
 's/double g = scale \* (exp(zv - lse\[n\])/double g = scale * (exp(zv - lse[0])/'  # wrong index
)
fail=0
for m in "${muts[@]}"; do
  cp /tmp/oracle_orig.c oracle/cce_oracle.c
  sed -i "$m" oracle/cce_oracle.c
  if cmp -s /tmp/oracle_orig.c oracle/cce_oracle.c; then echo "NO-OP mutation: $m"; fail=1; continue; fi
  python -c "import oracle; oracle.build(force=True)"
  if python -m pytest tests/test_oracle_pins.py -q -x >/dev/null 2>&1; then
    echo "SURVIVED: $m"; fail=1
  else
    echo "killed:   $m"
  fi
done
exit $fail
