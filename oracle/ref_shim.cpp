// placeholder: filled in with the reference control-plane shim
