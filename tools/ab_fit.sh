#!/bin/bash
# A/B the fit (route geometry + terminal field) of library variants
for lib in "$@"; do printf "%s " $lib; ECO_B200_LIB=$lib python tools/fit_probe.py | tail -1; done
