#!/bin/bash
# usage: tools/sass_fn.sh object pattern  -> SASS of the first function whose mangled name matches
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '/Function : /{p = ($0 ~ pat)} p && /^[ \t]+\/\*[0-9a-f]{4,5}\*\//{print}' | sed 's/^\s*//; s/\/\*[0-9a-fx]*\*\/\s*$//'
