"""Reference-side bindings of libhbrelu.so."""
