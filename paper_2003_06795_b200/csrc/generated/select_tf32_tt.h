#ifndef SELECT_TF32_TT_H
#define SELECT_TF32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tt_config;

static inline select_tf32_tt_config select_tf32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(1087)) {
        if (m < INT64_C(8870)) {
            if (n < INT64_C(287)) {
                if (m < INT64_C(1109)) {
                    if (k < INT64_C(992)) {
                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(555)) {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(544)) {
                        if (n < INT64_C(79)) {
                            if (k < INT64_C(118)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(28)) {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(314)) {
                                        if (n < INT64_C(46)) {
                                            if (m < INT64_C(2218)) {
                                                if (k < INT64_C(167)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(4435)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(167)) {
                                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(768)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (k < INT64_C(405)) {
                        if (m < INT64_C(1109)) {
                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(182)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(992)) {
                            if (m < INT64_C(448)) {
                                if (m < INT64_C(139)) {
                                    if (m < INT64_C(70)) {
                                        if (k < INT64_C(702)) {
                                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(702)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(702)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(1025)) {
                                if (m < INT64_C(278)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(393)) {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(28)) {
                if (m < INT64_C(35480)) {
                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(91)) {
                        if (k < INT64_C(168)) {
                            if (k < INT64_C(96)) {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(146)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(384)) {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(384)) {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(91)) {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(1432)) {
            if (m < INT64_C(555)) {
                if (n < INT64_C(363)) {
                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(139)) {
                        if (m < INT64_C(12)) {
                            if (k < INT64_C(2897)) {
                                if (k < INT64_C(1620)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(3)) {
                                        if (m < INT64_C(2)) {
                                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                if (k < INT64_C(2897)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(28)) {
                                        select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(3072)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(2173)) {
                    if (m < INT64_C(35480)) {
                        if (m < INT64_C(8870)) {
                            if (m < INT64_C(2218)) {
                                select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(182)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (n < INT64_C(182)) {
                                    select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(363)) {
                            select_tf32_tt_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
            return out;
        }
    }
}

#endif /* SELECT_TF32_TT_H */
